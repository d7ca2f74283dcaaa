// Shared helpers for the sm_100a kernels of the BH t-SNE hot path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "bhtsne_b200.h"

namespace bh {

// Records a message in the thread-local error slot; returns `code`.
int set_error(int code, const char *fmt, ...);
// Maps a CUDA error to BH_ERR_CUDA with a message (or BH_OK).
int cuda_status(cudaError_t e, const char *what);

constexpr int kSMs = 148;  // B200

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Warp-wide butterfly sum: every lane ends with the bit-identical value.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// GPU-scope relaxed accesses for flag+value words (decoupled look-back).
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ void st_relaxed(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v));
}

// Block-level exclusive prefix sum of one value per thread (blockDim <= 1024,
// multiple of 32).  `smem` needs 32 entries.  Returns the exclusive prefix;
// *total receives the block total.
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T *smem, T *total) {
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const unsigned nwarps = blockDim.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (unsigned)o) x += y;
    }
    if (lane == 31) smem[warp] = x;
    __syncthreads();
    if (warp == 0) {
        T w = lane < nwarps ? smem[lane] : T(0);
        T s = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= (unsigned)o) s += y;
        }
        if (lane < nwarps) smem[lane] = s - w;  // exclusive warp offsets
        if (lane == 31) *total = s;
    }
    __syncthreads();
    T r = smem[warp] + x - v;
    __syncthreads();
    return r;
}

}  // namespace bh

#define BH_CHECK_LAUNCH(what)                                                 \
    do {                                                                      \
        cudaError_t e_ = cudaGetLastError();                                  \
        if (e_ != cudaSuccess) return bh::cuda_status(e_, what);              \
    } while (0)

#define BH_REQUIRE(cond, ...)                                                 \
    do {                                                                      \
        if (!(cond)) return bh::set_error(BH_ERR_ARG, __VA_ARGS__);           \
    } while (0)

static inline cudaStream_t bh_cs(bh_stream_t s) { return (cudaStream_t)s; }
static inline size_t bh_align(size_t x) { return (x + 255) & ~(size_t)255; }
static inline int bh_blocks(int64_t n, int per) {
    int64_t b = (n + per - 1) / per;
    return (int)(b < 1 ? 1 : b);
}
