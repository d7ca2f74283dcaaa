// Shared helpers for the sm_100a kernels of the BH t-SNE hot path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <utility>

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

// ---------------------------------------------------------------------------
// Point precision (the reference's run dtype, io.py:21-30): T = float (f32
// storage, f32 pair math) or double (f64 storage and arithmetic).
// ---------------------------------------------------------------------------
template <typename T> struct P2;
template <> struct P2<float> { using type = float2; };
template <> struct P2<double> { using type = double2; };
template <typename T> using p2_t = typename P2<T>::type;

template <typename T> __device__ __forceinline__ p2_t<T> mk2(T a, T b);
template <> __device__ __forceinline__ float2 mk2<float>(float a, float b) {
    return make_float2(a, b);
}
template <> __device__ __forceinline__ double2 mk2<double>(double a, double b) {
    return make_double2(a, b);
}

// Node records (include/bhtsne_b200.h): f32 trees use one 16-B word
// {com.x, com.y, mass, info}; f64 trees two, {com.x, com.y} (f64) then
// {mass, info, 0, 0}.
template <typename T> struct NodeRec;
// f32 records hold the point count as a float (exact below 2^24 points;
// the f32 traversal weighs a cell by float(mass) in any case), so the
// traversal reads its weight without a conversion per child
template <> struct NodeRec<float> {
    static constexpr int kWords = 1;
    __device__ static void store(void *base, int64_t i, float2 c, uint32_t m,
                                 uint32_t info) {
        ((float4 *)base)[i] = make_float4(c.x, c.y, __uint2float_rn(m),
                                          __uint_as_float(info));
    }
    __device__ static void store_info(void *base, int64_t i, uint32_t info) {
        ((float4 *)base)[i].w = __uint_as_float(info);
    }
    __device__ static uint32_t info(const void *base, int64_t i) {
        return __float_as_uint(((const float4 *)base)[i].w);
    }
    __device__ static uint32_t mass(const void *base, int64_t i) {
        return __float2uint_rn(((const float4 *)base)[i].z);
    }
    __device__ static float2 com(const void *base, int64_t i) {
        const float4 r = ((const float4 *)base)[i];
        return make_float2(r.x, r.y);
    }
};
template <> struct NodeRec<double> {
    static constexpr int kWords = 2;
    __device__ static void store(void *base, int64_t i, double2 c, uint32_t m,
                                 uint32_t info) {
        ((double2 *)base)[2 * i] = c;
        ((uint4 *)base)[2 * i + 1] = make_uint4(m, info, 0u, 0u);
    }
    __device__ static void store_info(void *base, int64_t i, uint32_t info) {
        ((uint4 *)base)[2 * i + 1].y = info;
    }
    __device__ static uint32_t info(const void *base, int64_t i) {
        return ((const uint4 *)base)[2 * i + 1].y;
    }
    __device__ static uint32_t mass(const void *base, int64_t i) {
        return ((const uint4 *)base)[2 * i + 1].x;
    }
    __device__ static double2 com(const void *base, int64_t i) {
        return ((const double2 *)base)[2 * i];
    }
};

}  // namespace bh

// Device-side checks of a debug build (-DBH_DEBUG, tools/build_variant.py):
// compute-sanitizer is unavailable on this GPU pool, so the kernels' own
// invariants (traversal stack bounds, node indices, share ranges) trap.
#ifdef BH_DEBUG
#include <cstdio>
#define BH_DASSERT(c)                                                         \
    do {                                                                      \
        if (!(c)) {                                                           \
            printf("BH_DASSERT failed %s:%d: %s\n", __FILE__, __LINE__, #c);  \
            __trap();                                                         \
        }                                                                     \
    } while (0)
#else
#define BH_DASSERT(c) \
    do {              \
    } while (0)
#endif

#define BH_CHECK_LAUNCH(what)                                           \
    do {                                                                      \
        cudaError_t e_ = cudaGetLastError();                                  \
        if (e_ != cudaSuccess) return bh::cuda_status(e_, what);              \
    } while (0)

#define BH_REQUIRE(cond, ...)                                                 \
    do {                                                                      \
        if (!(cond)) return bh::set_error(BH_ERR_ARG, __VA_ARGS__);           \
    } while (0)

static inline cudaStream_t bh_cs(bh_stream_t s) { return (cudaStream_t)s; }

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL) along the iteration's kernel chain: a
// kernel launched with bh_launch may be scheduled while its predecessor in
// the stream is still finishing; it calls bh_pdl_wait() before touching the
// predecessor's results (griddepcontrol.wait, a no-op without a programmatic
// dependency) and bh_pdl_trigger() to let its own successor launch early.
// Captured into CUDA graphs as programmatic edges.  BH_PDL=0 disables it.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void bh_pdl_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void bh_pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;");
}

static inline bool bh_pdl_enabled() {
    static const bool on = [] {
        const char *s = getenv("BH_PDL");
        return s ? atoi(s) != 0 : true;
    }();
    return on;
}

// Which kernels take a programmatic dependency on their predecessor
// (tuning knob BH_PDL_KERNELS: comma-separated name prefixes; "all"/"none").
// Measured at C3 (it/s): none 484.3, all 482.5, summarize levels only 486.3
// -- within noise; on for the summarize chain only (its 11 short launches).
static inline bool bh_pdl_for(const char *what) {
    static const char *list = [] {
        const char *s = getenv("BH_PDL_KERNELS");
        return s ? s : "k_summarize";
    }();
    if (!bh_pdl_enabled()) return false;
    if (!strcmp(list, "all")) return true;
    for (const char *p = list; *p;) {
        const char *e = strchr(p, ',');
        const size_t len = e ? (size_t)(e - p) : strlen(p);
        if (len && !strncmp(what, p, len)) return true;
        if (!e) break;
        p = e + 1;
    }
    return false;
}

template <typename... KArgs, typename... Args>
static inline cudaError_t bh_launch(const char *what, void (*kernel)(KArgs...),
                                    dim3 grid, dim3 block, size_t smem,
                                    cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = bh_pdl_for(what) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

#define BH_LAUNCH(what, kernel, grid, block, smem, st, ...)                   \
    do {                                                                      \
        cudaError_t e_ = bh_launch(what, kernel, dim3(grid), dim3(block), smem, st, \
                                   __VA_ARGS__);                              \
        if (e_ != cudaSuccess) return bh::cuda_status(e_, what);              \
    } while (0)
static inline size_t bh_align(size_t x) { return (x + 255) & ~(size_t)255; }
static inline int bh_blocks(int64_t n, int per) {
    int64_t b = (n + per - 1) / per;
    return (int)(b < 1 ? 1 : b);
}
