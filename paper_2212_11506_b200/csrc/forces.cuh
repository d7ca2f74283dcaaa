// Helpers shared by the f32 (forces.cu) and f64 (forces_f64.cu) force
// kernels: launch shape, warp primitives, streaming loads and the
// GPU-count-invariant Z reduction.
#pragma once

#include "common.cuh"

namespace bh {

#ifndef BH_REP_WARPS
// 4 warps per traversal CTA at 9 CTAs/SM (56 registers, no spills): the
// fused force pass interleaves traversal and sweep CTAs more finely than
// with 8-warp CTAs (1.705 vs 1.775 ms at C3 iteration 600)
#define BH_REP_WARPS 4
#endif
constexpr int kRepWarps = BH_REP_WARPS;
constexpr int kRepThreads = kRepWarps * 32;
static_assert(kRepThreads == BH_REP_POINTS_PER_PARTIAL,
              "one Z partial per traversal CTA (include/bhtsne_b200.h)");

static inline int rep_grid(int64_t npts) { return bh_blocks(npts, kRepThreads); }

// Deterministic warp reduction: lane-strided sequential partials, then a
// butterfly.  Called by one full warp; every lane returns the total.
__device__ __forceinline__ double fixed_sum(const double *x, int64_t n) {
    double s = 0.0;
    for (int64_t i = threadIdx.x & 31; i < n; i += 32) s = __dadd_rn(s, __ldcg(&x[i]));
    return warp_sum(s);
}

// Deterministic fold of n f64 partials by one CTA of kFoldThreads: thread t
// sums x[t], x[t + kFoldThreads], ... in order, a butterfly per warp, then
// the warps in order.  The engine's Z total on one GPU (bh_step_zsum's
// tail) and after the all-reduce on several (bh_sum_partials) -- the same
// fold, so Z is bitwise independent of the GPU count.  Result valid in
// thread 0.
constexpr int kFoldThreads = 256;
__device__ __forceinline__ double cta_fold(const double *x, int64_t n,
                                           double *s_w /* kFoldThreads/32 */) {
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += kFoldThreads)
        s = __dadd_rn(s, __ldcg(&x[i]));
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = s;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kFoldThreads / 32; w++) t = __dadd_rn(t, s_w[w]);
    return t;
}

// The row range of a CSR sweep: explicit, or the engine's share (bh_part_t):
// rows [part->lo, part->split) when which == 0 (the side-stream sweep),
// [part->split, part->hi) otherwise.
template <typename Args>
__device__ __forceinline__ void att_rows(const Args &A, int64_t &b, int64_t &e) {
    if (A.part) {
        b = A.which ? A.part->split : A.part->lo;
        e = A.which ? A.part->hi : A.part->split;
    } else {
        b = A.row_begin;
        e = A.row_end;
    }
}

struct RepCounts {
    int internal, leafnodes, leafpts, accepted;
};

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ int4 ld_stream_i4(const int32_t *p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

__device__ __forceinline__ float4 ld_stream_f4(const float *p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}

__device__ __forceinline__ double2 ld_stream_d2(const double *p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                 : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}

// Full-warp ballot; the traversal keeps the whole warp converged (every
// branch is warp-uniform), so no divergence check is needed around it.
__device__ __forceinline__ uint32_t ballot_full(bool p) {
    uint32_t r;
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t"
        "vote.sync.ballot.b32 %0, q, 0xffffffff;\n\t}"
        : "=r"(r) : "r"((uint32_t)p));
    return r;
}

struct Acc64 {
    double z, r0, r1;
};

// Z: per-CTA partial (128 points in Morton order), then one fixed-order
// warp reduction over all CTA partials (fixed_sum) -- the same reduction the
// multi-GPU path applies to the gathered partials, so Z is bitwise
// independent of the GPU count.  No CTA-wide barrier: the
// last warp of the CTA to finish folds the warp partials.  s_z has
// kRepWarps entries; *s_done starts at 0.
// zidx: this CTA's partial slot (its block index, or slot / 128 in the
// engine's slot mode); nblk: the CTAs that write partials [0, nblk).
__device__ __forceinline__ void rep_z_tail(double z, int warp, int lane,
                                           int64_t zidx, int64_t nblk,
                                           double *s_z, unsigned *s_done,
                                           double *zblock, unsigned *ticket,
                                           double *z_out) {
    const double wz = warp_sum(z);
    unsigned last = 0;
    if (lane == 0) {
        s_z[warp] = wz;
        __threadfence_block();
        last = atomicAdd(s_done, 1u) == kRepWarps - 1;
    }
    if (!__shfl_sync(0xffffffffu, last, 0)) return;
    __threadfence_block();
    if (lane == 0) {
        double bz = 0.0;
        for (int w = 0; w < kRepWarps; w++)
            bz = __dadd_rn(bz, ((volatile double *)s_z)[w]);
        zblock[zidx] = bz;
        if (z_out) {
            __threadfence();
            last = atomicAdd(ticket, 1u) == (unsigned)(nblk - 1);
        } else {
            last = 0;
        }
    }
    if (!__shfl_sync(0xffffffffu, last, 0)) return;
    __threadfence();
    const double tot = fixed_sum(zblock, nblk);
    if (lane == 0) {
        *z_out = tot;
        *ticket = 0;
    }
}

}  // namespace bh
