// Staged CSR sweep (forces.py:56-72): P is static between relabels, so each
// block of rows_per_block consecutive rows gets, once per relabel, the
// sorted list of the distinct columns its entries name (bh_attr_stage_build)
// and every entry a 16-bit slot into that list.  The sweep CTA of a block
// gathers its distinct y_j ONCE into shared memory (a gather of sorted,
// distinct columns touches few 128-B lines) and the entries then read y_j by
// slot from shared memory: the L1 data-pipe wavefronts of the per-entry
// global gathers (~22 lines per 32-lane gather at C3) -- the bound of the
// plain sweep -- become shared-memory reads.  The lanes,
// entries and summation order are those of k_attractive, so the result is
// bitwise the same.
#include <algorithm>

#include "forces.cuh"

namespace bh {

// ---- builder ---------------------------------------------------------------
// One CTA per row block (persistent over blocks).  The distinct columns are
// found with a bitmap in shared memory over a window of kWinBits columns
// (several windows when n is larger), ranked by a prefix popcount: the list
// is sorted by column by construction.
constexpr int kStageThreads = 1024;
constexpr int kGroupsPerThread = 11;               // groups of 4 words
constexpr int kWinGroups = kStageThreads * kGroupsPerThread;
constexpr int kWinWords = kWinGroups * 4;          // 45056 words = 176 KB
constexpr int64_t kWinBits = (int64_t)kWinWords * 32;  // 1,441,792 columns
constexpr size_t kStageSmem = (size_t)kWinWords * 4 + (size_t)kWinGroups * 2;
constexpr int kNoSlot = 0xFFFF;

__global__ void __launch_bounds__(kStageThreads, 1)
k_attr_stage_build(const int64_t *__restrict__ rp,
                   const int32_t *__restrict__ col, int64_t n, int R, int S,
                   int64_t nblocks, int32_t *__restrict__ ucol,
                   int32_t *__restrict__ ucount,
                   uint16_t *__restrict__ slot) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t *bm = (uint32_t *)smem_raw;
    uint16_t *rank4 = (uint16_t *)(bm + kWinWords);
    __shared__ int s_scan[32];
    __shared__ int s_total;
    const int tid = threadIdx.x;
    for (int w = tid; w < kWinWords; w += kStageThreads) bm[w] = 0u;
    __syncthreads();
    for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
        const int64_t r0 = b * R, r1 = min(r0 + (int64_t)R, n);
        const int64_t e0 = rp[r0], e1 = rp[r1];
        int ubase = 0;
        for (int64_t wlo = 0; wlo < n; wlo += kWinBits) {
            for (int64_t q = e0 + tid; q < e1; q += kStageThreads) {
                const int64_t c = (int64_t)col[q] - wlo;
                if (c >= 0 && c < kWinBits)
                    atomicOr(&bm[c >> 5], 1u << (c & 31));
            }
            __syncthreads();
            const int g0 = tid * kGroupsPerThread;
            int cnt = 0;
#pragma unroll
            for (int g = 0; g < kGroupsPerThread; g++) {
                const uint4 w4 = ((const uint4 *)bm)[g0 + g];
                cnt += __popc(w4.x) + __popc(w4.y) + __popc(w4.z) + __popc(w4.w);
            }
            int total;
            int run = ubase + block_exclusive_scan(cnt, s_scan, &s_total);
            total = s_total;
            for (int g = 0; g < kGroupsPerThread; g++) {
                rank4[g0 + g] = (uint16_t)min(run, kNoSlot);
                for (int j = 0; j < 4; j++) {
                    const int w = (g0 + g) * 4 + j;
                    uint32_t bits = bm[w];
                    while (bits) {
                        const int bit = __ffs(bits) - 1;
                        bits &= bits - 1;
                        if (run < S)
                            ucol[b * S + run] =
                                (int32_t)(wlo + (int64_t)w * 32 + bit);
                        run++;
                    }
                }
            }
            __syncthreads();
            for (int64_t q = e0 + tid; q < e1; q += kStageThreads) {
                const int64_t c = (int64_t)col[q] - wlo;
                if (c >= 0 && c < kWinBits) {
                    const int w = (int)(c >> 5), g = w >> 2;
                    int s = rank4[g];
                    for (int j = g * 4; j < w; j++) s += __popc(bm[j]);
                    s += __popc(bm[w] & ((1u << (c & 31)) - 1u));
                    slot[q] = (uint16_t)(s < S ? s : kNoSlot);
                }
            }
            __syncthreads();
            for (int g = 0; g < kGroupsPerThread; g++)
                ((uint4 *)bm)[g0 + g] = make_uint4(0u, 0u, 0u, 0u);
            ubase += total;
            __syncthreads();
        }
        if (tid == 0) ucount[b] = min(ubase, S);
    }
}

// ---- sweep -----------------------------------------------------------------
struct StagedArgs {
    const int64_t *__restrict__ rp;
    const int32_t *__restrict__ col;
    const float *__restrict__ val;
    const uint16_t *__restrict__ slot;
    const int32_t *__restrict__ ucol;
    const int32_t *__restrict__ ucount;
    int R, S;
    const float2 *__restrict__ y;
    int64_t row_begin, row_end;
    float exag_param;
    const bh_sched_t *__restrict__ sched;
    float2 *__restrict__ attr;
    const bh_part_t *__restrict__ part;
    int which;
};

__device__ __forceinline__ uint2 ld_stream_u2(const uint16_t *p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}

template <int G, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
k_attractive_staged(const StagedArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2 *ys = (float2 *)smem_raw;
    __shared__ int s_next;
    int64_t row_begin, row_end;
    att_rows(A, row_begin, row_end);
    const int R = A.R, S = A.S;
    const int64_t b = row_begin / R + blockIdx.x;
    const int64_t rlo = max(b * R, row_begin);
    const int64_t rhi = min((b + 1) * R, row_end);
    if (rlo >= rhi) return;
    const float2 *__restrict__ y = A.y;
    {
        const int nu = A.ucount[b];
        const int32_t *__restrict__ uc = A.ucol + b * S;
        for (int i = threadIdx.x; i < nu; i += THREADS) ys[i] = __ldg(&y[uc[i]]);
    }
    if (threadIdx.x == 0) s_next = 0;
    __syncthreads();
    const bh_sched_t *__restrict__ sched = A.sched;
    const float exag = sched ? (sched->iteration < sched->exaggeration_iters
                                    ? sched->exaggeration
                                    : 1.0f)
                             : A.exag_param;
    const int gl = threadIdx.x % G;
    const int lane = threadIdx.x & 31;
    constexpr int kRowsPerWarp = 32 / G;
    for (;;) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&s_next, kRowsPerWarp);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (rlo + base >= rhi) break;
        const int64_t row = rlo + base + lane / G;
        const bool ok = row < rhi;
        int64_t s = 0, e = 0;
        float2 yi = make_float2(0.f, 0.f);
        if (ok) {
            s = A.rp[row];
            e = A.rp[row + 1];
            yi = y[row];
        }
        double a0 = 0.0, a1 = 0.0;
#define BH_ATTR_TERM(YJ, V)                                                   \
    {                                                                         \
        float dx = yi.x - YJ.x, dy = yi.y - YJ.y;                             \
        float pq = __fmul_rn(V, exag) * rcp_approx(1.0f + dx * dx + dy * dy); \
        fx += pq * dx;                                                        \
        fy += pq * dy;                                                        \
    }
        const uint16_t *__restrict__ sp = A.slot + s;
        const int32_t *__restrict__ cp = A.col + s;
        const float *__restrict__ vp = A.val + s;
        const int len = (int)(e - s);
        for (int k = 4 * gl; k < len; k += 4 * G) {
            const uint2 sl = ld_stream_u2(sp + k);
            const float4 v = ld_stream_f4(vp + k);
            const unsigned s0 = sl.x & 0xFFFFu, s1 = sl.x >> 16;
            const unsigned s2 = sl.y & 0xFFFFu, s3 = sl.y >> 16;
            float2 y0, y1, y2, y3;
            if (max(max(s0, s1), max(s2, s3)) != (unsigned)kNoSlot) {
                y0 = ys[s0];
                y1 = ys[s1];
                y2 = ys[s2];
                y3 = ys[s3];
            } else {  // a column beyond the block's staged list
                y0 = s0 != (unsigned)kNoSlot ? ys[s0] : __ldg(&y[cp[k]]);
                y1 = s1 != (unsigned)kNoSlot ? ys[s1] : __ldg(&y[cp[k + 1]]);
                y2 = s2 != (unsigned)kNoSlot ? ys[s2] : __ldg(&y[cp[k + 2]]);
                y3 = s3 != (unsigned)kNoSlot ? ys[s3] : __ldg(&y[cp[k + 3]]);
            }
            float fx = 0.f, fy = 0.f;
            BH_ATTR_TERM(y0, v.x)
            BH_ATTR_TERM(y1, v.y)
            BH_ATTR_TERM(y2, v.z)
            BH_ATTR_TERM(y3, v.w)
            a0 += (double)fx;
            a1 += (double)fy;
        }
#undef BH_ATTR_TERM
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            a0 += __shfl_xor_sync(0xffffffffu, a0, o);
            a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        }
        if (ok && gl == 0) A.attr[row] = make_float2((float)a0, (float)a1);
    }
}

template <int THREADS, int MINB>
static int launch_staged(const StagedArgs &A, int grid, cudaStream_t st) {
    auto k = k_attractive_staged<16, THREADS, MINB>;
    const size_t smem = (size_t)A.S * sizeof(float2);
    static size_t set = 0;
    if (smem > set) {
        cudaError_t e = cudaFuncSetAttribute(
            k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return cuda_status(e, "k_attractive_staged smem");
        set = smem;
    }
    BH_LAUNCH("k_attractive_staged", k, grid, THREADS, smem, st, A);
    BH_CHECK_LAUNCH("k_attractive_staged");
    return BH_OK;
}

static int staged_dispatch(const StagedArgs &A, int grid, cudaStream_t st) {
    static const int threads = [] {
        const char *s = getenv("BH_STAGE_THREADS");
        return s ? atoi(s) : 512;
    }();
    switch (threads) {
    case 256: return launch_staged<256, 2>(A, grid, st);
    case 1024: return launch_staged<1024, 1>(A, grid, st);
    default: return launch_staged<512, 2>(A, grid, st);
    }
}

}  // namespace bh

using namespace bh;

extern "C" int bh_attr_stage_build(const int64_t *row_ptr, const int32_t *col,
                                   int64_t n, int rows_per_block, int slots,
                                   int32_t *ucol, int32_t *ucount,
                                   uint16_t *slot, bh_stream_t stream) {
    BH_REQUIRE(row_ptr && col && ucol && ucount && slot, "null argument");
    BH_REQUIRE(rows_per_block >= 1, "rows_per_block must be >= 1");
    BH_REQUIRE(slots >= 1 && slots <= kNoSlot - 128,
               "slots must be in [1, %d]", kNoSlot - 128);
    if (n <= 0) return BH_OK;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(
            k_attr_stage_build, cudaFuncAttributeMaxDynamicSharedMemorySize,
            (int)kStageSmem);
        if (e != cudaSuccess) return cuda_status(e, "k_attr_stage_build smem");
        attr_set = true;
    }
    const int64_t nblocks = (n + rows_per_block - 1) / rows_per_block;
    const int grid = (int)std::min<int64_t>(nblocks, kSMs);
    BH_LAUNCH("k_attr_stage_build", k_attr_stage_build, grid, kStageThreads,
              kStageSmem, bh_cs(stream), row_ptr, col, n, rows_per_block,
              slots, nblocks, ucol, ucount, slot);
    BH_CHECK_LAUNCH("k_attr_stage_build");
    return BH_OK;
}

extern "C" int bh_attractive_staged(const int64_t *row_ptr, const int32_t *col,
                                    const float *val, const uint16_t *slot,
                                    const int32_t *ucol, const int32_t *ucount,
                                    int rows_per_block, int slots,
                                    const float *y, int64_t row_begin,
                                    int64_t row_end, float exaggeration,
                                    const bh_sched_t *sched, float *attr,
                                    bh_stream_t stream) {
    BH_REQUIRE(row_ptr && col && val && slot && ucol && ucount && y && attr,
               "null argument");
    BH_REQUIRE(row_begin >= 0 && row_begin <= row_end, "bad row range");
    if (row_end == row_begin) return BH_OK;
    const StagedArgs A{row_ptr, col, val, slot, ucol, ucount, rows_per_block,
                       slots, (const float2 *)y, row_begin, row_end,
                       exaggeration, sched, (float2 *)attr, nullptr, 0};
    const int grid = (int)((row_end - 1) / rows_per_block
                           - row_begin / rows_per_block + 1);
    return staged_dispatch(A, grid, bh_cs(stream));
}

extern "C" int bh_step_attractive_staged(
    const int64_t *row_ptr, const int32_t *col, const float *val,
    const uint16_t *slot, const int32_t *ucol, const int32_t *ucount,
    int rows_per_block, int slots, const float *y, const bh_part_t *part,
    int64_t max_rows, const bh_sched_t *sched, float *attr,
    bh_stream_t stream) {
    BH_REQUIRE(part && sched, "part and sched are required");
    if (max_rows <= 0) return BH_OK;
    const StagedArgs A{row_ptr, col, val, slot, ucol, ucount, rows_per_block,
                       slots, (const float2 *)y, 0, 0, 1.0f, sched,
                       (float2 *)attr, part, 0};
    // rows [lo, split): at most max_rows of them, starting anywhere in a block
    const int grid = (int)((max_rows + rows_per_block - 1) / rows_per_block + 1);
    return staged_dispatch(A, grid, bh_cs(stream));
}
