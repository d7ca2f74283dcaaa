// Point-parallel kernels: bounds (quadtree.py:133-153), Morton codes
// (quadtree.py:156-185), the momentum/gains update with re-centering
// (optimizer.py:161-168, 195-224) and the centering pass.
//
// Bit-exactness: bounds and quantisation are computed in f64 with explicit
// round-to-nearest intrinsics (no FMA contraction);
// the update uses explicit f32 intrinsics in numpy's (NEP 50) operation order.
#include <float.h>

#include "common.cuh"

namespace bh {

constexpr int kPtThreads = 256;
constexpr int kPtMaxBlocks = kSMs * 8;

__device__ __forceinline__ uint32_t spread16(uint32_t x) {
    x &= 0xFFFFu;
    x = (x | (x << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}

__device__ __forceinline__ uint64_t spread32(uint64_t m) {  // _spread_bits
    m &= 0x00000000FFFFFFFFull;
    m = (m | (m << 16)) & 0x0000FFFF0000FFFFull;
    m = (m | (m << 8)) & 0x00FF00FF00FF00FFull;
    m = (m | (m << 4)) & 0x0F0F0F0F0F0F0F0Full;
    m = (m | (m << 2)) & 0x3333333333333333ull;
    m = (m | (m << 1)) & 0x5555555555555555ull;
    return m;
}

// compute_bounds (quadtree.py:145-153) from exact f32 extrema, plus the
// Morton constants of _morton_kernel (quadtree.py:179-181).
__device__ void finalize_bounds(float mn0, float mx0, float mn1, float mx1,
                                int nonfinite, int code_bits, float sh0,
                                float sh1, bh_bounds_t *out) {
    double dmn0 = mn0, dmx0 = mx0, dmn1 = mn1, dmx1 = mx1;
    double c0 = __dmul_rn(0.5, __dadd_rn(dmn0, dmx0));
    double c1 = __dmul_rn(0.5, __dadd_rn(dmn1, dmx1));
    double h0 = __dsub_rn(dmx0, c0), h1 = __dsub_rn(dmx1, c1);
    double half = h0 >= h1 ? h0 : h1;
    if (half <= 0.0) {
        double m = 1.0;
        if (fabs(c0) > m) m = fabs(c0);
        if (fabs(c1) > m) m = fabs(c1);
        half = __dmul_rn(1e-9, m);
    }
    double r = __dmul_rn(half, __dadd_rn(1.0, 1e-12));
    out->c0 = c0;
    out->c1 = c1;
    out->r_span = r;
    out->root0 = __dsub_rn(c0, r);
    out->root1 = __dsub_rn(c1, r);
    out->scale = __ddiv_rn(code_bits == 64 ? 2147483648.0 : 32768.0, r);
    out->shift0 = sh0;
    out->shift1 = sh1;
    out->nonfinite = nonfinite;
    out->code_bits = code_bits;
}

struct MinMax {
    float mn0, mx0, mn1, mx1;
    int bad;
};

__device__ __forceinline__ void mm_init(MinMax &m) {
    m.mn0 = m.mn1 = FLT_MAX;
    m.mx0 = m.mx1 = -FLT_MAX;
    m.bad = 0;
}

__device__ __forceinline__ void mm_add(MinMax &m, float a, float b) {
    if (!isfinite(a) || !isfinite(b)) m.bad = 1;
    m.mn0 = fminf(m.mn0, a);
    m.mx0 = fmaxf(m.mx0, a);
    m.mn1 = fminf(m.mn1, b);
    m.mx1 = fmaxf(m.mx1, b);
}

__device__ __forceinline__ void mm_warp(MinMax &m) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        m.mn0 = fminf(m.mn0, __shfl_xor_sync(0xffffffffu, m.mn0, o));
        m.mx0 = fmaxf(m.mx0, __shfl_xor_sync(0xffffffffu, m.mx0, o));
        m.mn1 = fminf(m.mn1, __shfl_xor_sync(0xffffffffu, m.mn1, o));
        m.mx1 = fmaxf(m.mx1, __shfl_xor_sync(0xffffffffu, m.mx1, o));
        m.bad |= __shfl_xor_sync(0xffffffffu, m.bad, o);
    }
}

// Block reduction of MinMax (and optionally two f64 sums); result valid in
// thread 0.
struct PtPartial {
    float4 mm;
    double s0, s1;
    int bad;
    int pad;
};

__device__ void block_reduce(MinMax m, double s0, double s1, PtPartial *out) {
    __shared__ MinMax sm[kPtThreads / 32];
    __shared__ double ss0[kPtThreads / 32], ss1[kPtThreads / 32];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    mm_warp(m);
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    if (l == 0) {
        sm[w] = m;
        ss0[w] = s0;
        ss1[w] = s1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        MinMax r = sm[0];
        double a = ss0[0], b = ss1[0];
        for (int i = 1; i < kPtThreads / 32; i++) {
            r.mn0 = fminf(r.mn0, sm[i].mn0);
            r.mx0 = fmaxf(r.mx0, sm[i].mx0);
            r.mn1 = fminf(r.mn1, sm[i].mn1);
            r.mx1 = fmaxf(r.mx1, sm[i].mx1);
            r.bad |= sm[i].bad;
            a = __dadd_rn(a, ss0[i]);
            b = __dadd_rn(b, ss1[i]);
        }
        out->mm = make_float4(r.mn0, r.mx0, r.mn1, r.mx1);
        out->s0 = a;
        out->s1 = b;
        out->bad = r.bad;
    }
}

// Last-block-done: returns true in the block that finishes last (all threads).
__device__ bool last_block(unsigned *ticket) {
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    return s_last;
}

// Fixed-order reduction of the per-block partials by the whole (last)
// block: thread i folds partials i, i+blockDim, ... in order, then the same
// fixed warp/block tree as block_reduce.  Deterministic for a given n (the
// grid is a function of n).  Result valid in thread 0.
__device__ PtPartial reduce_partials(const PtPartial *part, int nparts) {
    MinMax m;
    mm_init(m);
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
        float4 q = __ldcg(&part[i].mm);
        m.mn0 = fminf(m.mn0, q.x);
        m.mx0 = fmaxf(m.mx0, q.y);
        m.mn1 = fminf(m.mn1, q.z);
        m.mx1 = fmaxf(m.mx1, q.w);
        m.bad |= __ldcg(&part[i].bad);
        a = __dadd_rn(a, __ldcg(&part[i].s0));
        b = __dadd_rn(b, __ldcg(&part[i].s1));
    }
    __shared__ PtPartial s_r;
    block_reduce(m, a, b, &s_r);
    __syncthreads();
    return s_r;
}

__global__ void __launch_bounds__(kPtThreads)
k_bounds(const float2 *__restrict__ y, int64_t n, int code_bits,
         bh_bounds_t *out, PtPartial *part, unsigned *ticket) {
    MinMax m;
    mm_init(m);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float2 p = y[i];
        mm_add(m, p.x, p.y);
    }
    block_reduce(m, 0.0, 0.0, &part[blockIdx.x]);
    if (!last_block(ticket)) return;
    PtPartial r = reduce_partials(part, gridDim.x);
    if (threadIdx.x == 0) {
        finalize_bounds(r.mm.x, r.mm.y, r.mm.z, r.mm.w, r.bad, code_bits,
                        0.0f, 0.0f, out);
        *ticket = 0;
    }
}

template <int BITS>
__global__ void __launch_bounds__(kPtThreads)
k_morton(float2 *__restrict__ y, int64_t n, const bh_bounds_t *__restrict__ b,
         int apply_shift,
         typename std::conditional<BITS == 32, uint32_t, uint64_t>::type
             *__restrict__ codes) {
    const double root0 = b->root0, root1 = b->root1, scale = b->scale;
    const float sh0 = b->shift0, sh1 = b->shift1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float2 p = y[i];
        if (apply_shift) {
            p.x = __fsub_rn(p.x, sh0);
            p.y = __fsub_rn(p.y, sh1);
            y[i] = p;
        }
        double q0 = __dmul_rn(__dsub_rn((double)p.x, root0), scale);
        double q1 = __dmul_rn(__dsub_rn((double)p.y, root1), scale);
        if constexpr (BITS == 32) {
            uint32_t m0 = __double2uint_rz(q0), m1 = __double2uint_rz(q1);
            codes[i] = spread16(m0) | (spread16(m1) << 1);
        } else {
            uint64_t m0 = __double2ull_rz(q0), m1 = __double2ull_rz(q1);
            codes[i] = spread32(m0) | (spread32(m1) << 1);
        }
    }
}

__device__ __forceinline__ float sgnf(float x) {
    return (float)((x > 0.0f) - (x < 0.0f));
}

// One coordinate of _update_coord (optimizer.py:161-168) in numpy f32
// semantics: every Python scalar is cast to float32, no FMA contraction.
__device__ __forceinline__ void update_coord(float &y, float &v, float &g,
                                             float grad, float mom, float lr,
                                             float mg) {
    bool flip = sgnf(grad) != sgnf(v);
    float gn = flip ? __fadd_rn(g, 0.2f) : __fmul_rn(g, 0.8f);
    gn = gn < mg ? mg : gn;
    g = gn;
    float vn = __fsub_rn(__fmul_rn(mom, v), __fmul_rn(__fmul_rn(lr, gn), grad));
    v = vn;
    y = __fadd_rn(y, vn);
}

__global__ void __launch_bounds__(kPtThreads)
k_update(float2 *__restrict__ y, float2 *__restrict__ v,
         float2 *__restrict__ g, const float2 *__restrict__ attr,
         const float2 *__restrict__ rep, const int32_t *__restrict__ rep_rank,
         int64_t n, bh_sched_t *sched, bh_bounds_t *out, int code_bits,
         PtPartial *part, unsigned *ticket) {
    const int it = sched->iteration;
    const float zf = __double2float_rn(sched->z);
    const float mom = it < sched->momentum_switch ? sched->momentum_early
                                                  : sched->momentum_late;
    const float lr = sched->learning_rate, mg = sched->min_gain;
    MinMax m;
    mm_init(m);
    double s0 = 0.0, s1 = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float2 a = attr[i], r = rep[rep_rank ? (int64_t)rep_rank[i] : i];
        // grad = 4.0 * (attr - rep / z)   (optimizer.py:205-207)
        float gx = __fmul_rn(4.0f, __fsub_rn(a.x, __fdiv_rn(r.x, zf)));
        float gy = __fmul_rn(4.0f, __fsub_rn(a.y, __fdiv_rn(r.y, zf)));
        if (!isfinite(gx) || !isfinite(gy))
            atomicMin((unsigned long long *)&sched->bad,
                      ((unsigned long long)(unsigned)it << 32) |
                          (unsigned long long)i);
        float2 yy = y[i], vv = v[i], gg = g[i];
        update_coord(yy.x, vv.x, gg.x, gx, mom, lr, mg);
        update_coord(yy.y, vv.y, gg.y, gy, mom, lr, mg);
        y[i] = yy;
        v[i] = vv;
        g[i] = gg;
        mm_add(m, yy.x, yy.y);
        s0 = __dadd_rn(s0, (double)yy.x);
        s1 = __dadd_rn(s1, (double)yy.y);
    }
    block_reduce(m, s0, s1, &part[blockIdx.x]);
    if (!last_block(ticket)) return;
    PtPartial r = reduce_partials(part, gridDim.x);
    if (threadIdx.x == 0) {
        // y -= f32(mean_f64(y))   (optimizer.py:220-221); rounding is
        // monotone, so min(y - m) == f32(min(y) - m): the bounds of the
        // re-centred cloud come straight from the extrema.
        float m0 = __double2float_rn(__ddiv_rn(r.s0, (double)n));
        float m1 = __double2float_rn(__ddiv_rn(r.s1, (double)n));
        finalize_bounds(__fsub_rn(r.mm.x, m0), __fsub_rn(r.mm.y, m0),
                        __fsub_rn(r.mm.z, m1), __fsub_rn(r.mm.w, m1), r.bad,
                        code_bits, m0, m1, out);
        sched->iteration = it + 1;
        *ticket = 0;
    }
}

__global__ void k_center(float2 *__restrict__ y, int64_t n,
                         const bh_bounds_t *__restrict__ b) {
    const float sh0 = b->shift0, sh1 = b->shift1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float2 p = y[i];
        p.x = __fsub_rn(p.x, sh0);
        p.y = __fsub_rn(p.y, sh1);
        y[i] = p;
    }
}

static int pt_grid(int64_t n) {
    int b = bh_blocks(n, kPtThreads);
    return b < kPtMaxBlocks ? b : kPtMaxBlocks;
}

static size_t pt_ws_bytes(int64_t n) {
    return bh_align(sizeof(PtPartial) * pt_grid(n)) + 256;
}

}  // namespace bh

using namespace bh;

extern "C" size_t bh_bounds_workspace_bytes(int64_t n) { return pt_ws_bytes(n); }
extern "C" size_t bh_update_workspace_bytes(int64_t n) { return pt_ws_bytes(n); }

extern "C" int bh_bounds(const float *y, int64_t n, int code_bits,
                         bh_bounds_t *out, void *ws, size_t ws_bytes,
                         bh_stream_t stream) {
    BH_REQUIRE(n >= 1, "need at least one point");
    BH_REQUIRE(code_bits == 32 || code_bits == 64, "code_bits must be 32 or 64");
    BH_REQUIRE(ws_bytes >= pt_ws_bytes(n), "bounds workspace too small");
    int grid = pt_grid(n);
    char *w = (char *)ws;
    PtPartial *part = (PtPartial *)w;
    unsigned *ticket = (unsigned *)(w + bh_align(sizeof(PtPartial) * grid));
    k_bounds<<<grid, kPtThreads, 0, bh_cs(stream)>>>((const float2 *)y, n,
                                                     code_bits, out, part,
                                                     ticket);
    BH_CHECK_LAUNCH("k_bounds");
    return BH_OK;
}

extern "C" int bh_morton(float *y, int64_t n, const bh_bounds_t *bounds,
                         int code_bits, int apply_shift, void *codes,
                         bh_stream_t stream) {
    BH_REQUIRE(n >= 1, "need at least one point");
    int grid = pt_grid(n);
    if (code_bits == 32)
        k_morton<32><<<grid, kPtThreads, 0, bh_cs(stream)>>>(
            (float2 *)y, n, bounds, apply_shift, (uint32_t *)codes);
    else if (code_bits == 64)
        k_morton<64><<<grid, kPtThreads, 0, bh_cs(stream)>>>(
            (float2 *)y, n, bounds, apply_shift, (uint64_t *)codes);
    else
        return set_error(BH_ERR_UNSUPPORTED, "code_bits must be 32 or 64");
    BH_CHECK_LAUNCH("k_morton");
    return BH_OK;
}

extern "C" int bh_update(float *y, float *v, float *g, const float *attr,
                         const float *rep, const int32_t *rep_rank, int64_t n,
                         bh_sched_t *sched,
                         bh_bounds_t *bounds_out, int code_bits, void *ws,
                         size_t ws_bytes, bh_stream_t stream) {
    BH_REQUIRE(n >= 1, "need at least one point");
    BH_REQUIRE(ws_bytes >= pt_ws_bytes(n), "update workspace too small");
    int grid = pt_grid(n);
    char *w = (char *)ws;
    PtPartial *part = (PtPartial *)w;
    unsigned *ticket = (unsigned *)(w + bh_align(sizeof(PtPartial) * grid));
    k_update<<<grid, kPtThreads, 0, bh_cs(stream)>>>(
        (float2 *)y, (float2 *)v, (float2 *)g, (const float2 *)attr,
        (const float2 *)rep, rep_rank, n, sched, bounds_out, code_bits, part,
        ticket);
    BH_CHECK_LAUNCH("k_update");
    return BH_OK;
}

extern "C" int bh_center(float *y, int64_t n, const bh_bounds_t *bounds,
                         bh_stream_t stream) {
    k_center<<<pt_grid(n), kPtThreads, 0, bh_cs(stream)>>>((float2 *)y, n,
                                                           bounds);
    BH_CHECK_LAUNCH("k_center");
    return BH_OK;
}

// ---------------------------------------------------------------------------
// Row gather / scatter / permutation inverse (relabeling plumbing).
// ---------------------------------------------------------------------------
namespace bh {

template <typename T>
__global__ void k_gather(const T *__restrict__ src, const int32_t *__restrict__ idx,
                         int64_t n, T *__restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}

template <typename T>
__global__ void k_scatter(const T *__restrict__ src, const int32_t *__restrict__ idx,
                          int64_t n, T *__restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[idx[i]] = src[i];
}

__global__ void k_invert(const int32_t *__restrict__ perm, int64_t n,
                         int32_t *__restrict__ inv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        inv[perm[i]] = (int32_t)i;
}

}  // namespace bh

extern "C" int bh_gather_rows(const void *src, const int32_t *idx, int64_t n,
                              int elem_bytes, void *dst, bh_stream_t stream) {
    const int grid = pt_grid(n);
    cudaStream_t st = bh_cs(stream);
    if (elem_bytes == 4)
        k_gather<uint32_t><<<grid, kPtThreads, 0, st>>>((const uint32_t *)src, idx, n, (uint32_t *)dst);
    else if (elem_bytes == 8)
        k_gather<uint2><<<grid, kPtThreads, 0, st>>>((const uint2 *)src, idx, n, (uint2 *)dst);
    else
        return set_error(BH_ERR_ARG, "elem_bytes must be 4 or 8");
    BH_CHECK_LAUNCH("k_gather");
    return BH_OK;
}

extern "C" int bh_scatter_rows(const void *src, const int32_t *idx, int64_t n,
                               int elem_bytes, void *dst, bh_stream_t stream) {
    const int grid = pt_grid(n);
    cudaStream_t st = bh_cs(stream);
    if (elem_bytes == 4)
        k_scatter<uint32_t><<<grid, kPtThreads, 0, st>>>((const uint32_t *)src, idx, n, (uint32_t *)dst);
    else if (elem_bytes == 8)
        k_scatter<uint2><<<grid, kPtThreads, 0, st>>>((const uint2 *)src, idx, n, (uint2 *)dst);
    else
        return set_error(BH_ERR_ARG, "elem_bytes must be 4 or 8");
    BH_CHECK_LAUNCH("k_scatter");
    return BH_OK;
}

extern "C" int bh_invert_perm(const int32_t *perm, int64_t n, int32_t *inv,
                              bh_stream_t stream) {
    k_invert<<<pt_grid(n), kPtThreads, 0, bh_cs(stream)>>>(perm, n, inv);
    BH_CHECK_LAUNCH("k_invert");
    return BH_OK;
}
