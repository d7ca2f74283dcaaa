// Point-parallel kernels: bounds (quadtree.py:133-153), Morton codes
// (quadtree.py:156-185), the momentum/gains update with re-centering
// (optimizer.py:161-168, 195-224) and the centering pass.
//
// Bit-exactness: bounds and quantisation are computed in f64 with explicit
// round-to-nearest intrinsics (no FMA contraction);
// the update uses explicit f32 intrinsics in numpy's (NEP 50) operation order.
#include <float.h>

#include <type_traits>

#include "keys.cuh"

namespace bh {

constexpr int kPtThreads = 256;
#ifndef BH_PT_BLOCKS_PER_SM
#define BH_PT_BLOCKS_PER_SM 4  // update 26 us vs 28 (8), 34 (16)
#endif
constexpr int kPtMaxBlocks = kSMs * BH_PT_BLOCKS_PER_SM;

// compute_bounds (quadtree.py:145-153) from exact f32 extrema, plus the
// Morton constants of _morton_kernel (quadtree.py:179-181).
// Extrema arrive as f64 (exact for f32 points); sh*: the pending shift in
// the run precision (f32 fields for f32 runs, f64 fields for f64 runs).
__device__ void finalize_bounds(double dmn0, double dmx0, double dmn1,
                                double dmx1, int nonfinite, int code_bits,
                                float sh0, float sh1, double sh0d, double sh1d,
                                bh_bounds_t *out) {
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
    out->shift0_f64 = sh0d;
    out->shift1_f64 = sh1d;
}

template <typename T>
struct MinMax {
    T mn0, mx0, mn1, mx1;
    int bad;
};

template <typename T> __device__ __forceinline__ T t_max();
template <> __device__ __forceinline__ float t_max<float>() { return FLT_MAX; }
template <> __device__ __forceinline__ double t_max<double>() { return DBL_MAX; }

template <typename T>
__device__ __forceinline__ void mm_init(MinMax<T> &m) {
    m.mn0 = m.mn1 = t_max<T>();
    m.mx0 = m.mx1 = -t_max<T>();
    m.bad = 0;
}

template <typename T>
__device__ __forceinline__ void mm_add(MinMax<T> &m, T a, T b) {
    if (!isfinite(a) || !isfinite(b)) m.bad = 1;
    m.mn0 = fmin(m.mn0, a);
    m.mx0 = fmax(m.mx0, a);
    m.mn1 = fmin(m.mn1, b);
    m.mx1 = fmax(m.mx1, b);
}

template <typename T>
__device__ __forceinline__ void mm_warp(MinMax<T> &m) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        m.mn0 = fmin(m.mn0, __shfl_xor_sync(0xffffffffu, m.mn0, o));
        m.mx0 = fmax(m.mx0, __shfl_xor_sync(0xffffffffu, m.mx0, o));
        m.mn1 = fmin(m.mn1, __shfl_xor_sync(0xffffffffu, m.mn1, o));
        m.mx1 = fmax(m.mx1, __shfl_xor_sync(0xffffffffu, m.mx1, o));
        m.bad |= __shfl_xor_sync(0xffffffffu, m.bad, o);
    }
}

// Block reduction of MinMax (and optionally two f64 sums); result valid in
// thread 0.
template <typename T>
struct PtPartial {
    T mn0, mx0, mn1, mx1;
    double s0, s1;
    int bad;
    int pad;
};

template <typename T>
__device__ void block_reduce(MinMax<T> m, double s0, double s1,
                             PtPartial<T> *out) {
    __shared__ MinMax<T> sm[kPtThreads / 32];
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
        MinMax<T> r = sm[0];
        double a = ss0[0], b = ss1[0];
        for (int i = 1; i < kPtThreads / 32; i++) {
            r.mn0 = fmin(r.mn0, sm[i].mn0);
            r.mx0 = fmax(r.mx0, sm[i].mx0);
            r.mn1 = fmin(r.mn1, sm[i].mn1);
            r.mx1 = fmax(r.mx1, sm[i].mx1);
            r.bad |= sm[i].bad;
            a = __dadd_rn(a, ss0[i]);
            b = __dadd_rn(b, ss1[i]);
        }
        out->mn0 = r.mn0;
        out->mx0 = r.mx0;
        out->mn1 = r.mn1;
        out->mx1 = r.mx1;
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
template <typename T>
__device__ PtPartial<T> reduce_partials(const PtPartial<T> *part, int nparts) {
    MinMax<T> m;
    mm_init(m);
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
        m.mn0 = fmin(m.mn0, __ldcg(&part[i].mn0));
        m.mx0 = fmax(m.mx0, __ldcg(&part[i].mx0));
        m.mn1 = fmin(m.mn1, __ldcg(&part[i].mn1));
        m.mx1 = fmax(m.mx1, __ldcg(&part[i].mx1));
        m.bad |= __ldcg(&part[i].bad);
        a = __dadd_rn(a, __ldcg(&part[i].s0));
        b = __dadd_rn(b, __ldcg(&part[i].s1));
    }
    __shared__ PtPartial<T> s_r;
    block_reduce(m, a, b, &s_r);
    __syncthreads();
    return s_r;
}

template <typename T>
__global__ void __launch_bounds__(kPtThreads)
k_bounds(const p2_t<T> *__restrict__ y, int64_t n, int code_bits,
         bh_bounds_t *out, PtPartial<T> *part, unsigned *ticket) {
    bh_pdl_trigger();  // the successor may launch early (PDL)
    bh_pdl_wait();     // the predecessor's results are visible

    MinMax<T> m;
    mm_init(m);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const p2_t<T> p = y[i];
        mm_add(m, p.x, p.y);
    }
    block_reduce(m, 0.0, 0.0, &part[blockIdx.x]);
    if (!last_block(ticket)) return;
    PtPartial<T> r = reduce_partials(part, gridDim.x);
    if (threadIdx.x == 0) {
        finalize_bounds(r.mn0, r.mx0, r.mn1, r.mx1, r.bad, code_bits, 0.0f,
                        0.0f, 0.0, 0.0, out);
        *ticket = 0;
    }
}

#ifndef BH_HILBERT_LUT
// Hilbert keys four levels per shared-memory table lookup (keys.cuh); 0
// keeps the level-by-level walk (A/B builds)
#define BH_HILBERT_LUT 1
#endif
template <int BITS, typename T, bool HILBERT = false>
__global__ void __launch_bounds__(kPtThreads)
k_morton(p2_t<T> *__restrict__ y, int64_t n, const bh_bounds_t *__restrict__ b,
         int apply_shift,
         typename std::conditional<BITS == 32, uint32_t, uint64_t>::type
             *__restrict__ codes) {
    bh_pdl_trigger();  // the successor may launch early (PDL)
    bh_pdl_wait();     // the predecessor's results are visible

    __shared__ uint16_t s_lut[HILBERT && BH_HILBERT_LUT ? 1024 : 1];
    if (HILBERT && BH_HILBERT_LUT) hilbert_lut_load(s_lut);
    const double root0 = b->root0, root1 = b->root1, scale = b->scale;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        p2_t<T> p = y[i];
        if (apply_shift) {
            p = shifted(p, b);
            y[i] = p;
        }
        if (HILBERT && BH_HILBERT_LUT)
            codes[i] = point_key_hilbert_lut<BITS>((double)p.x, (double)p.y,
                                                   root0, root1, scale, s_lut);
        else
            codes[i] = point_key<BITS, HILBERT>((double)p.x, (double)p.y,
                                                root0, root1, scale);
    }
}

__device__ __forceinline__ float sgnf(float x) {
    return (float)((x > 0.0f) - (x < 0.0f));
}

// One coordinate of _update_coord (optimizer.py:161-168) in numpy f32
// semantics: every Python scalar is cast to float32, no FMA contraction.
__device__ __forceinline__ double sgnd(double x) {
    return (double)((x > 0.0) - (x < 0.0));
}

__device__ __forceinline__ void update_coord(double &y, double &v, double &g,
                                             double grad, double mom,
                                             double lr, double mg) {
    // the same operations on float64 arrays (f64 run mode)
    bool flip = sgnd(grad) != sgnd(v);
    double gn = flip ? __dadd_rn(g, 0.2) : __dmul_rn(g, 0.8);
    gn = gn < mg ? mg : gn;
    g = gn;
    double vn = __dsub_rn(__dmul_rn(mom, v), __dmul_rn(__dmul_rn(lr, gn), grad));
    v = vn;
    y = __dadd_rn(y, vn);
}

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

// Schedule constants and gradient in the run precision: f32 runs use the
// f32 fields and f32(Z) (numpy's weak-scalar promotion of rep / z on f32
// arrays), f64 runs the f64 fields and Z itself.
struct SchedF32 {
    float z, mom, lr, mg;
    __device__ void init(const bh_sched_t *s, int it) {
        z = __double2float_rn(s->z);
        mom = it < s->momentum_switch ? s->momentum_early : s->momentum_late;
        lr = s->learning_rate;
        mg = s->min_gain;
    }
    __device__ float grad(float a, float r) const {
        return __fmul_rn(4.0f, __fsub_rn(a, __fdiv_rn(r, z)));
    }
};
struct SchedF64 {
    double z, mom, lr, mg;
    __device__ void init(const bh_sched_t *s, int it) {
        z = s->z;
        mom = it < s->momentum_switch ? s->momentum_early_f64
                                      : s->momentum_late_f64;
        lr = s->learning_rate_f64;
        mg = s->min_gain_f64;
    }
    __device__ double grad(double a, double r) const {
        return __dmul_rn(4.0, __dsub_rn(a, __ddiv_rn(r, z)));
    }
};
template <typename T>
using sched_t = typename std::conditional<std::is_same<T, float>::value,
                                          SchedF32, SchedF64>::type;

__device__ __forceinline__ float fsub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double fsub_rn(double a, double b) { return __dsub_rn(a, b); }

// The last block of k_update / k_finish: y -= T(mean_f64(y))
// (optimizer.py:220-221) is published as the pending shift; rounding is
// monotone, so min(y - m) == rn(min(y) - m) and the bounds of the re-centred
// cloud come straight from the extrema.  Advances the iteration.
template <typename T>
__device__ void finish_iteration(const PtPartial<T> *part, int nparts,
                                 int64_t n, int it, int code_bits,
                                 bh_sched_t *sched, bh_bounds_t *out,
                                 unsigned *ticket) {
    PtPartial<T> r = reduce_partials(part, nparts);
    if (threadIdx.x == 0) {
        const double d0 = __ddiv_rn(r.s0, (double)n);
        const double d1 = __ddiv_rn(r.s1, (double)n);
        const T m0 = (T)d0, m1 = (T)d1;
        finalize_bounds(fsub_rn(r.mn0, m0), fsub_rn(r.mx0, m0),
                        fsub_rn(r.mn1, m1), fsub_rn(r.mx1, m1), r.bad,
                        code_bits, (float)m0, (float)m1, (double)m0,
                        (double)m1, out);
        sched->iteration = it + 1;
        *ticket = 0;
    }
}

// The update of slots [lo, hi) (all n points, or the engine's share `pr`).
// reduce: also reduce the new y (extrema and f64 sums, grid-stride order
// over [0, n)) and finish the iteration -- one GPU, where [lo, hi) = [0, n).
// Otherwise (several GPUs) k_finish does that after the y exchange, over
// the same grid in the same order, so the mean and the bounds are bitwise
// those of one GPU.  ysend (optional): the new y of the share, packed from 0.
template <typename T>
__global__ void __launch_bounds__(kPtThreads)
k_update(p2_t<T> *__restrict__ y, p2_t<T> *__restrict__ v,
         p2_t<T> *__restrict__ g, const p2_t<T> *__restrict__ attr,
         const p2_t<T> *__restrict__ rep, const int32_t *__restrict__ rep_rank,
         int64_t n, bh_sched_t *sched, bh_bounds_t *out, int code_bits,
         PtPartial<T> *part, unsigned *ticket,
         const bh_part_t *__restrict__ pr, p2_t<T> *__restrict__ ysend,
         int reduce) {
    bh_pdl_trigger();  // the successor may launch early (PDL)
    bh_pdl_wait();     // the predecessor's results are visible

    const int it = sched->iteration;
    sched_t<T> S;
    S.init(sched, it);
    MinMax<T> m;
    mm_init(m);
    double s0 = 0.0, s1 = 0.0;
    const int64_t lo = pr ? pr->lo : 0, hi = pr ? pr->hi : n;
    for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
         i < hi; i += (int64_t)gridDim.x * blockDim.x) {
        const p2_t<T> a = attr[i], r = rep[rep_rank ? (int64_t)rep_rank[i] : i];
        // grad = 4.0 * (attr - rep / z)   (optimizer.py:205-207)
        const T gx = S.grad(a.x, r.x), gy = S.grad(a.y, r.y);
        if (!isfinite(gx) || !isfinite(gy))
            atomicMin((unsigned long long *)&sched->bad,
                      ((unsigned long long)(unsigned)it << 32) |
                          (unsigned long long)i);
        p2_t<T> yy = y[i], vv = v[i], gg = g[i];
        update_coord(yy.x, vv.x, gg.x, gx, S.mom, S.lr, S.mg);
        update_coord(yy.y, vv.y, gg.y, gy, S.mom, S.lr, S.mg);
        y[i] = yy;
        v[i] = vv;
        g[i] = gg;
        if (ysend) ysend[i - lo] = yy;
        mm_add(m, yy.x, yy.y);
        s0 = __dadd_rn(s0, (double)yy.x);
        s1 = __dadd_rn(s1, (double)yy.y);
    }
    if (!reduce) return;
    block_reduce(m, s0, s1, &part[blockIdx.x]);
    if (!last_block(ticket)) return;
    finish_iteration(part, gridDim.x, n, it, code_bits, sched, out, ticket);
}

// The reduction half of k_update over the exchanged y (several GPUs).
template <typename T>
__global__ void __launch_bounds__(kPtThreads)
k_finish(const p2_t<T> *__restrict__ y, int64_t n, bh_sched_t *sched,
         bh_bounds_t *out, int code_bits, PtPartial<T> *part,
         unsigned *ticket) {
    bh_pdl_trigger();
    bh_pdl_wait();
    const int it = sched->iteration;
    MinMax<T> m;
    mm_init(m);
    double s0 = 0.0, s1 = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const p2_t<T> yy = y[i];
        mm_add(m, yy.x, yy.y);
        s0 = __dadd_rn(s0, (double)yy.x);
        s1 = __dadd_rn(s1, (double)yy.y);
    }
    block_reduce(m, s0, s1, &part[blockIdx.x]);
    if (!last_block(ticket)) return;
    finish_iteration(part, gridDim.x, n, it, code_bits, sched, out, ticket);
}

template <typename T>
__global__ void k_center(p2_t<T> *__restrict__ y, int64_t n,
                         const bh_bounds_t *__restrict__ b) {
    bh_pdl_trigger();  // the successor may launch early (PDL)
    bh_pdl_wait();     // the predecessor's results are visible

    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = shifted(y[i], b);
}

static int pt_grid(int64_t n) {
    int b = bh_blocks(n, kPtThreads);
    return b < kPtMaxBlocks ? b : kPtMaxBlocks;
}

static size_t pt_ws_bytes(int64_t n) {
    return bh_align(sizeof(PtPartial<double>) * pt_grid(n)) + 256;
}

template <typename T>
static int bounds_impl(const T *y, int64_t n, int code_bits, bh_bounds_t *out,
                       void *ws, size_t ws_bytes, bh_stream_t stream) {
    BH_REQUIRE(n >= 1, "need at least one point");
    BH_REQUIRE(code_bits == 32 || code_bits == 64, "code_bits must be 32 or 64");
    BH_REQUIRE(ws_bytes >= pt_ws_bytes(n), "bounds workspace too small");
    int grid = pt_grid(n);
    char *w = (char *)ws;
    PtPartial<T> *part = (PtPartial<T> *)w;
    unsigned *ticket = (unsigned *)(w + bh_align(sizeof(PtPartial<T>) * grid));
    BH_LAUNCH("k_bounds", k_bounds<T>, grid, kPtThreads, 0, bh_cs(stream),
              (const p2_t<T> *)y, n, code_bits, out, part, ticket);
    return BH_OK;
}

template <typename T, bool HILBERT = false>
static int morton_impl(T *y, int64_t n, const bh_bounds_t *bounds,
                       int code_bits, int apply_shift, void *codes,
                       bh_stream_t stream) {
    BH_REQUIRE(n >= 1, "need at least one point");
    int grid = pt_grid(n);
    if (code_bits == 32)
        BH_LAUNCH("k_morton", (k_morton<32, T, HILBERT>), grid, kPtThreads, 0,
                  bh_cs(stream), (p2_t<T> *)y, n, bounds, apply_shift,
                  (uint32_t *)codes);
    else if (code_bits == 64)
        BH_LAUNCH("k_morton", (k_morton<64, T, HILBERT>), grid, kPtThreads, 0,
                  bh_cs(stream), (p2_t<T> *)y, n, bounds, apply_shift,
                  (uint64_t *)codes);
    else
        return set_error(BH_ERR_UNSUPPORTED, "code_bits must be 32 or 64");
    return BH_OK;
}

template <typename T>
static int update_impl(T *y, T *v, T *g, const T *attr, const T *rep,
                       const int32_t *rep_rank, int64_t n, bh_sched_t *sched,
                       bh_bounds_t *bounds_out, int code_bits, void *ws,
                       size_t ws_bytes, bh_stream_t stream) {
    BH_REQUIRE(n >= 1, "need at least one point");
    BH_REQUIRE(ws_bytes >= pt_ws_bytes(n), "update workspace too small");
    int grid = pt_grid(n);
    char *w = (char *)ws;
    PtPartial<T> *part = (PtPartial<T> *)w;
    unsigned *ticket = (unsigned *)(w + bh_align(sizeof(PtPartial<T>) * grid));
    BH_LAUNCH("k_update", k_update<T>, grid, kPtThreads, 0, bh_cs(stream),
              (p2_t<T> *)y, (p2_t<T> *)v, (p2_t<T> *)g, (const p2_t<T> *)attr,
              (const p2_t<T> *)rep, rep_rank, n, sched, bounds_out, code_bits,
              part, ticket, (const bh_part_t *)nullptr, (p2_t<T> *)nullptr, 1);
    return BH_OK;
}

template <typename T>
static int step_update_impl(T *y, T *v, T *g, const T *attr, const T *rep,
                            const bh_part_t *pr, int64_t n, bh_sched_t *sched,
                            bh_bounds_t *bounds_out, int code_bits,
                            int reduce, T *ysend, void *ws, size_t ws_bytes,
                            bh_stream_t stream) {
    BH_REQUIRE(n >= 1, "need at least one point");
    BH_REQUIRE(ws_bytes >= pt_ws_bytes(n), "update workspace too small");
    int grid = pt_grid(n);
    char *w = (char *)ws;
    PtPartial<T> *part = (PtPartial<T> *)w;
    unsigned *ticket = (unsigned *)(w + bh_align(sizeof(PtPartial<T>) * grid));
    BH_LAUNCH("k_update", k_update<T>, grid, kPtThreads, 0, bh_cs(stream),
              (p2_t<T> *)y, (p2_t<T> *)v, (p2_t<T> *)g, (const p2_t<T> *)attr,
              (const p2_t<T> *)rep, (const int32_t *)nullptr, n, sched,
              bounds_out, code_bits, part, ticket, pr, (p2_t<T> *)ysend,
              reduce);
    return BH_OK;
}

template <typename T>
static int step_finish_impl(const T *y, int64_t n, bh_sched_t *sched,
                            bh_bounds_t *bounds_out, int code_bits, void *ws,
                            size_t ws_bytes, bh_stream_t stream) {
    BH_REQUIRE(n >= 1, "need at least one point");
    BH_REQUIRE(ws_bytes >= pt_ws_bytes(n), "update workspace too small");
    int grid = pt_grid(n);
    char *w = (char *)ws;
    PtPartial<T> *part = (PtPartial<T> *)w;
    unsigned *ticket = (unsigned *)(w + bh_align(sizeof(PtPartial<T>) * grid));
    BH_LAUNCH("k_finish", k_finish<T>, grid, kPtThreads, 0, bh_cs(stream),
              (const p2_t<T> *)y, n, sched, bounds_out, code_bits, part,
              ticket);
    return BH_OK;
}

}  // namespace bh

using namespace bh;

extern "C" size_t bh_bounds_workspace_bytes(int64_t n) { return pt_ws_bytes(n); }
extern "C" size_t bh_update_workspace_bytes(int64_t n) { return pt_ws_bytes(n); }

extern "C" int bh_bounds(const float *y, int64_t n, int code_bits,
                         bh_bounds_t *out, void *ws, size_t ws_bytes,
                         bh_stream_t stream) {
    return bounds_impl(y, n, code_bits, out, ws, ws_bytes, stream);
}

extern "C" int bh_bounds_f64(const double *y, int64_t n, int code_bits,
                             bh_bounds_t *out, void *ws, size_t ws_bytes,
                             bh_stream_t stream) {
    return bounds_impl(y, n, code_bits, out, ws, ws_bytes, stream);
}

extern "C" int bh_morton(float *y, int64_t n, const bh_bounds_t *bounds,
                         int code_bits, int apply_shift, void *codes,
                         bh_stream_t stream) {
    return morton_impl(y, n, bounds, code_bits, apply_shift, codes, stream);
}

extern "C" int bh_morton_f64(double *y, int64_t n, const bh_bounds_t *bounds,
                             int code_bits, int apply_shift, void *codes,
                             bh_stream_t stream) {
    return morton_impl(y, n, bounds, code_bits, apply_shift, codes, stream);
}

extern "C" int bh_hilbert(float *y, int64_t n, const bh_bounds_t *bounds,
                          int code_bits, int apply_shift, void *codes,
                          bh_stream_t stream) {
    return morton_impl<float, true>(y, n, bounds, code_bits, apply_shift,
                                    codes, stream);
}

extern "C" int bh_hilbert_f64(double *y, int64_t n, const bh_bounds_t *bounds,
                              int code_bits, int apply_shift, void *codes,
                              bh_stream_t stream) {
    return morton_impl<double, true>(y, n, bounds, code_bits, apply_shift,
                                     codes, stream);
}

extern "C" int bh_update(float *y, float *v, float *g, const float *attr,
                         const float *rep, const int32_t *rep_rank, int64_t n,
                         bh_sched_t *sched, bh_bounds_t *bounds_out,
                         int code_bits, void *ws, size_t ws_bytes,
                         bh_stream_t stream) {
    return update_impl(y, v, g, attr, rep, rep_rank, n, sched, bounds_out,
                       code_bits, ws, ws_bytes, stream);
}

extern "C" int bh_update_f64(double *y, double *v, double *g,
                             const double *attr, const double *rep,
                             const int32_t *rep_rank, int64_t n,
                             bh_sched_t *sched, bh_bounds_t *bounds_out,
                             int code_bits, void *ws, size_t ws_bytes,
                             bh_stream_t stream) {
    return update_impl(y, v, g, attr, rep, rep_rank, n, sched, bounds_out,
                       code_bits, ws, ws_bytes, stream);
}

extern "C" int bh_step_update(float *y, float *v, float *g, const float *attr,
                              const float *rep, const bh_part_t *part,
                              int64_t n, bh_sched_t *sched,
                              bh_bounds_t *bounds_out, int code_bits,
                              int reduce, float *ysend, void *ws,
                              size_t ws_bytes, bh_stream_t stream) {
    return step_update_impl(y, v, g, attr, rep, part, n, sched, bounds_out,
                            code_bits, reduce, ysend, ws, ws_bytes, stream);
}

extern "C" int bh_step_update_f64(double *y, double *v, double *g,
                                  const double *attr, const double *rep,
                                  const bh_part_t *part, int64_t n,
                                  bh_sched_t *sched, bh_bounds_t *bounds_out,
                                  int code_bits, int reduce, double *ysend,
                                  void *ws, size_t ws_bytes,
                                  bh_stream_t stream) {
    return step_update_impl(y, v, g, attr, rep, part, n, sched, bounds_out,
                            code_bits, reduce, ysend, ws, ws_bytes, stream);
}

extern "C" int bh_step_finish(const float *y, int64_t n, bh_sched_t *sched,
                              bh_bounds_t *bounds_out, int code_bits,
                              void *ws, size_t ws_bytes, bh_stream_t stream) {
    return step_finish_impl(y, n, sched, bounds_out, code_bits, ws, ws_bytes,
                            stream);
}

extern "C" int bh_step_finish_f64(const double *y, int64_t n,
                                  bh_sched_t *sched, bh_bounds_t *bounds_out,
                                  int code_bits, void *ws, size_t ws_bytes,
                                  bh_stream_t stream) {
    return step_finish_impl(y, n, sched, bounds_out, code_bits, ws, ws_bytes,
                            stream);
}

extern "C" int bh_center(float *y, int64_t n, const bh_bounds_t *bounds,
                         bh_stream_t stream) {
    BH_LAUNCH("k_center", k_center<float>, pt_grid(n), kPtThreads, 0,
              bh_cs(stream), (float2 *)y, n, bounds);
    return BH_OK;
}

extern "C" int bh_center_f64(double *y, int64_t n, const bh_bounds_t *bounds,
                             bh_stream_t stream) {
    BH_LAUNCH("k_center", k_center<double>, pt_grid(n), kPtThreads, 0,
              bh_cs(stream), (double2 *)y, n, bounds);
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
    else if (elem_bytes == 16)
        k_gather<uint4><<<grid, kPtThreads, 0, st>>>((const uint4 *)src, idx, n, (uint4 *)dst);
    else
        return set_error(BH_ERR_ARG, "elem_bytes must be 4, 8 or 16");
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
    else if (elem_bytes == 16)
        k_scatter<uint4><<<grid, kPtThreads, 0, st>>>((const uint4 *)src, idx, n, (uint4 *)dst);
    else
        return set_error(BH_ERR_ARG, "elem_bytes must be 4, 8 or 16");
    BH_CHECK_LAUNCH("k_scatter");
    return BH_OK;
}

extern "C" int bh_invert_perm(const int32_t *perm, int64_t n, int32_t *inv,
                              bh_stream_t stream) {
    k_invert<<<pt_grid(n), kPtThreads, 0, bh_cs(stream)>>>(perm, n, inv);
    BH_CHECK_LAUNCH("k_invert");
    return BH_OK;
}
