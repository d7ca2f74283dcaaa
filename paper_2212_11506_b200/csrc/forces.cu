// Force kernels: Barnes-Hut repulsion (forces.py:85-150), attractive CSR
// sweep (forces.py:56-82), exact O(N^2) repulsion (forces.py:153-182) and
// the KL rows (optimizer.py:227-239).
#include <algorithm>
#include <type_traits>

#include "forces.cuh"

namespace bh {

// ---------------------------------------------------------------------------
// Repulsion: warp-synchronous BH traversal with per-lane acceptance masks.
//
// A warp owns 32 consecutive points in Morton order.  Its stack holds child
// GROUPS (the consecutive children of one opened node) plus the mask of
// lanes that opened that node.  Popping a group loads its <= 4 node records
// once for the whole warp (a broadcast of <= 64 contiguous bytes); every lane
// in the mask applies the reference's per-point rule to each child exactly
// as forces.py:99-128 does -- a leaf contributes its points directly (self
// skipped by index), an internal node is accepted iff (2r)^2 < theta^2 d^2,
// else that lane needs its children.  The children are pushed once with the
// ballot of the lanes that need them.  Each lane therefore visits exactly the
// node set of its own reference traversal (same accept decisions, same
// contributions); lanes that accepted or never reached a node idle for it.
// Pair math is f32; contributions of one popped group are summed in f32 and
// added to f64 accumulators.
// ---------------------------------------------------------------------------
// Per-pop context of a lane: its point, the group's R2 and whether the lane
// opened the node whose children are being visited.
#ifndef BH_R2_MASK
#define BH_R2_MASK 1
#endif

struct GroupCtx {
    const float4 *__restrict__ node;
    const float2 *__restrict__ ys;
    float2 yi;
    float r2;   // this lane's acceptance threshold (R2, or -1: not in the mask)
    float r2u;  // the group's R2 (pushed, quartered, with its children)
    bool mine;
    uint32_t self;
    int lane;
    uint32_t depth;  // of the group's children
};

// p ? x : 0 as one select on the f32 value (kept ahead of the f64
// conversion, which the compiler otherwise selects twice per double)
__device__ __forceinline__ float sel_f32(bool p, float x) {
    float r;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
        "selp.f32 %0, %1, 0f00000000, q;\n\t}"
        : "=f"(r) : "f"(x), "r"((uint32_t)p));
    return r;
}

// The m > 1 points [s, s + m) of a depth-D bucket leaf (coincident codes)
// for one lane (forces.py:102-110): loaded once per 32 and broadcast by
// shuffles; f32 partials per 32 points, then f64.  Self is skipped by index
// unless SC (its exact +1 to z is then subtracted at the end).
template <bool SC>
__device__ __forceinline__ void bh_bucket(const GroupCtx &g, uint32_t s,
                                          uint32_t m, Acc64 &a64) {
    for (uint32_t b = 0; b < m; b += 32) {
        const float2 pq = (b + g.lane < m) ? g.ys[s + b + g.lane]
                                           : make_float2(0.f, 0.f);
        const int nb = (int)min(32u, m - b);
        float bz = 0.f, bx = 0.f, by = 0.f;
        for (int jj = 0; jj < nb; jj++) {
            const float px = __shfl_sync(0xffffffffu, pq.x, jj);
            const float py = __shfl_sync(0xffffffffu, pq.y, jj);
            const float ex = g.yi.x - px, ey = g.yi.y - py;
            const float kk = rcp_approx(1.0f + fmaf(ex, ex, ey * ey));
            const float ww = (SC || s + b + jj != g.self) ? kk : 0.f;
            const float ww2 = ww * kk;
            bz += ww;
            bx = fmaf(ww2, ex, bx);
            by = fmaf(ww2, ey, by);
        }
        a64.z += (double)sel_f32(g.mine, bz);
        a64.r0 += (double)sel_f32(g.mine, bx);
        a64.r1 += (double)sel_f32(g.mine, by);
    }
}

// One child of a group above depth D for one lane (the reference rule,
// forces.py:99-128), where every leaf
// holds exactly one point (leaf iff count == 1 or depth == D,
// quadtree.py:262-300).  Leaf vs internal is folded into the predicates: a
// leaf is never approximated and its record is its point with mass 1, so
// it "accepts" unconditionally (minus self, compared by the whole info
// word); an internal node accepts iff d2 > R2.  Same decisions and
// contributions as the reference's per-point walk.
template <bool COUNT, bool SC, bool FIRST = false>
__device__ __forceinline__ uint32_t bh_child_fast(const GroupCtx &g,
                                                  const float4 r, float &fz,
                                                  float &fx, float &fy,
                                                  RepCounts &cn) {
    const uint32_t info = __float_as_uint(r.w);
    const float dx = g.yi.x - r.x, dy = g.yi.y - r.y;
    const float d2 = fmaf(dx, dx, dy * dy);
    const bool leaf = (int32_t)info < 0;
    const bool acc = leaf || d2 > g.r2;
    if (COUNT && g.mine) {
        if (leaf) {
            cn.leafnodes++;
            cn.leafpts += (int)r.z;
        } else {
            cn.internal++;
            cn.accepted += acc;
        }
    }
    // lanes outside the mask are zeroed once per group (bh_group); with SC
    // the self leaf is not tested here: it adds exactly k = 1/(1+0) = 1 to
    // z and 0 to the force, and rep_block subtracts that 1 (kScTheta)
    const bool use = acc && (SC || info != (BH_LEAF_BIT | g.self));
    const float w = use ? r.z : 0.f;  // the cell's point count
#if BH_R2_MASK
    // lanes outside the mask carry R2 = -1: they accept every child, so
    // they never ask for children (their sums are zeroed per group)
    const uint32_t need = ballot_full(!acc);
#else
    const uint32_t need = ballot_full(g.mine && !acc);
#endif
    const float k = rcp_approx(1.0f + d2);
    const float wk = w * k, wk2 = wk * k;
    if (FIRST) {  // the group's first term starts the partials (no 0 + x)
        fz = wk;
        fx = wk2 * dx;
        fy = wk2 * dy;
    } else {
        fz += wk;
        fx = fmaf(wk2, dx, fx);
        fy = fmaf(wk2, dy, fy);
    }
    return need;
}

// Visit the CNT consecutive children starting at `first` (a group above
// depth D), then push every child some lane must open in one lane-parallel
// step (lane c writes child c's entry; child 0 ends on top so the first
// subtree is popped first).
template <int CNT, bool COUNT, bool SC>
__device__ __forceinline__ void bh_group(const GroupCtx &g, uint32_t first,
                                         Acc64 &a64, RepCounts &cn,
                                         uint4 *stk, int &sp) {
    float4 rec[CNT];  // all loads issued up front (ILP)
    BH_DASSERT(first + CNT <= (uint32_t)BH_CHILD_MASK);
#pragma unroll
    for (int c = 0; c < CNT; c++) rec[c] = __ldg(&g.node[first + c]);
    float fz = 0.f, fx = 0.f, fy = 0.f;
    uint32_t pm[CNT], inf[CNT];
#pragma unroll
    for (int c = 0; c < CNT; c++) {
        inf[c] = __float_as_uint(rec[c].w);
        pm[c] = c == 0 ? bh_child_fast<COUNT, SC, true>(g, rec[c], fz, fx, fy, cn)
                       : bh_child_fast<COUNT, SC>(g, rec[c], fz, fx, fy, cn);
    }
    // out-of-mask lanes add nothing (exact zero, in f32)
    a64.z += (double)sel_f32(g.mine, fz);
    a64.r0 += (double)sel_f32(g.mine, fx);
    a64.r1 += (double)sel_f32(g.mine, fy);
    // lane c < CNT pushes child c's group if any lane must open it; one
    // ballot gives every writer its slot (child 0 ends on top)
    uint32_t info = inf[0], msk = pm[0];
#pragma unroll
    for (int c = 1; c < CNT; c++)
        if (g.lane == c) {
            info = inf[c];
            msk = pm[c];
        }
    const bool push = g.lane < CNT && msk != 0u;
    const uint32_t nz = ballot_full(push);
    if (push)
        stk[sp + __popc(nz >> (g.lane + 1))] = make_uint4(
            info, msk, __float_as_uint(g.r2u * 0.25f), g.depth + 1u);
    sp += __popc(nz);
}

// A group at depth D (max depth): every child is a leaf -- a single point
// or a coincident-code bucket (quadtree.py leaf rule) -- so there is no
// acceptance test, no ballot and nothing to push.
template <int CNT, bool COUNT, bool SC>
__device__ __forceinline__ void bh_group_leaves(const GroupCtx &g,
                                                uint32_t first, Acc64 &a64,
                                                RepCounts &cn) {
    float4 rec[CNT];
#pragma unroll
    for (int c = 0; c < CNT; c++) rec[c] = __ldg(&g.node[first + c]);
    float fz = 0.f, fx = 0.f, fy = 0.f;
#pragma unroll
    for (int c = 0; c < CNT; c++) {
        const uint32_t info = __float_as_uint(rec[c].w);
        const uint32_t m = __float2uint_rn(rec[c].z);
        if (COUNT && g.mine) {
            cn.leafnodes++;
            cn.leafpts += (int)m;
        }
        if (m > 1u) {  // bucket (warp-uniform)
            bh_bucket<SC>(g, info & ~BH_LEAF_BIT, m, a64);
        } else {
            const float dx = g.yi.x - rec[c].x, dy = g.yi.y - rec[c].y;
            const float k = rcp_approx(1.0f + fmaf(dx, dx, dy * dy));
            // self: exact test, or SC's +1 subtracted at the end
            const float w = (SC || info != (BH_LEAF_BIT | g.self)) ? k : 0.f;
            const float w2 = w * k;
            fz += w;
            fx = fmaf(w2, dx, fx);
            fy = fmaf(w2, dy, fy);
        }
    }
    a64.z += (double)sel_f32(g.mine, fz);
    a64.r0 += (double)sel_f32(g.mine, fx);
    a64.r1 += (double)sel_f32(g.mine, fy);
}

// Stack entry (16 B, one STS.128 / broadcast LDS.128): x = the opened
// node's info word (first child | (children - 1) << 29), y = mask of the
// lanes that opened it, z = R2 = side^2 / theta^2 of the children's cells
// (f32; exact quartering per level), w = the depth of those children.
struct RepArgs {
    const float4 *__restrict__ node;
    const float2 *__restrict__ ys;
    const int32_t *__restrict__ order;
    const float2 *__restrict__ y_query;
    const bh_bounds_t *__restrict__ bounds;
    const int32_t *__restrict__ status;
    double theta;
    int64_t t_begin, t_end;
    int sorted_out;
    float2 *__restrict__ rep;
    double *__restrict__ zpart;
    int4 *__restrict__ counts;
    double *__restrict__ zblock;
    unsigned *__restrict__ ticket;
    double *__restrict__ z_out;
    // engine mode (part != NULL): the share's hi - lo storage slots, taken
    // in the current Morton order -- qlist[i] (several GPUs: the share's
    // slots in sorted order, bh_step_qlist) or order[i] (one GPU: all of
    // them); coordinates y_query[slot] (ys[i] on one GPU), self = its sorted
    // position (rank[slot]); rep[slot] and zpart[slot]
    const bh_part_t *__restrict__ part;
    const int32_t *__restrict__ rank;
    const int32_t *__restrict__ qlist;
};

// Self correction (SC): when theta <= kScTheta no point accepts an
// ancestor of its own leaf -- d^2 <= (2 sqrt2 r)^2 = 8 r^2 for the point and
// the centre of mass inside one cell, while acceptance needs d^2 >
// 4 r^2 / theta^2 >= 8.16 r^2 -- so every point meets itself exactly once,
// in its own leaf (single-point or depth-D bucket), where the pair term is
// k = 1/(1+0) = 1 to z and 0 to the force.  No child or bucket point is
// then tested against self; rep_block subtracts the 1 at the end.  Above
// kScTheta the exact per-child / per-point self test stays.
#ifndef BH_SC_THETA
#define BH_SC_THETA 0.7  // (A/B builds: -1 turns the correction off)
#endif
constexpr double kScTheta = BH_SC_THETA;

#ifndef BH_REP_MIN_BLOCKS
// 9 CTAs x 4 warps per SM (56 registers).  With 8-warp CTAs: 5 per SM
// (48 registers) measured 1.23 ms vs 1.33 ms (4), 1.44 ms (3), 2.29 ms (6,
// heavy spills) at C3 iteration 600
#define BH_REP_MIN_BLOCKS 9
#endif

// CTA `bid` of the `nblk` traversal CTAs: points t_begin + 256 bid + [0, 256).
template <int D, bool COUNT, bool QUERY, bool SC>
__device__ __forceinline__ void rep_block(const RepArgs &A, int64_t bid,
                                          int64_t nblk) {
    constexpr int CAP = 3 * D + 2;
    __shared__ uint4 s_stack[kRepWarps][CAP];
    __shared__ double s_z[kRepWarps];
    __shared__ unsigned s_done;
    const float4 *__restrict__ node = A.node;
    const float2 *__restrict__ ys = A.ys;
    const int32_t *__restrict__ order = A.order;
    const int32_t *__restrict__ status = A.status;
    const bh_bounds_t *__restrict__ bounds = A.bounds;
    const int64_t t_begin = A.t_begin, t_end = A.t_end;
    const double theta = A.theta;
    double *__restrict__ zblock = A.zblock;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool slots = A.part != nullptr;
    const int64_t lo = slots ? 0 : t_begin;
    const int64_t hi = slots ? A.part->hi - A.part->lo : t_end;
    if (lo + bid * kRepThreads >= hi) return;  // engine mode: past the share
    if (threadIdx.x == 0) s_done = 0;
    __syncthreads();
    const int64_t t = lo + (bid * kRepWarps + warp) * 32 + lane;
    const bool valid = t < hi && *status == BH_OK;
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    float2 yi = make_float2(0.f, 0.f);
    uint32_t self = (uint32_t)t;
    int64_t slot = 0;
    if (valid) {
        if (slots && A.qlist) {
            slot = A.qlist[t];
            BH_DASSERT(slot >= A.part->lo && slot < A.part->hi);
            yi = A.y_query[slot];
            if (!SC) self = (uint32_t)A.rank[slot];
        } else if (slots) {
            slot = order[t];
            yi = ys[t];
        } else {
            yi = QUERY ? A.y_query[order[t]] : ys[t];
        }
    }
    double r0 = 0.0, r1 = 0.0, z = 0.0;
    RepCounts cn = {0, 0, 0, 0};
    uint4 *stk = s_stack[warp];
    Acc64 a{0.0, 0.0, 0.0};

    int sp = 0;
    if (act) {
        if (lane == 0) {
            // the root "group": node 0 alone; R2 = (2 r_span)^2 / theta^2
            // (+inf at theta = 0: nothing is ever accepted)
            const double side = 2.0 * bounds->r_span;
            const float r2root = (float)((side * side) / (theta * theta));
            stk[0] = make_uint4(0u, act, __float_as_uint(r2root), 0u);
        }
        sp = 1;
        __syncwarp();
    }
    while (sp > 0) {
        // (no barrier after the read: every lane's ballots below depend on
        // `ent`, so all reads complete before any lane overwrites the slot;
        // the barrier at the end of the loop orders the pushes before the
        // next read)
        BH_DASSERT(sp >= 1 && sp <= CAP);
        const uint4 ent = stk[--sp];
        const uint32_t first = ent.x & BH_CHILD_MASK;
        const bool mine = (ent.y >> lane) & 1u;
        const float r2u = __uint_as_float(ent.z);
#if BH_R2_MASK
        const float r2 = mine ? r2u : -1.0f;
#else
        const float r2 = r2u;
#endif
        const GroupCtx g{node, ys, yi, r2, r2u, mine, self, lane, ent.w};
        // straight-line code for the (warp-uniform) number of children;
        // the branch-free body above the deepest level (warp-uniform)
        if (ent.w < (uint32_t)D) {
            // most groups are full (4 children): test that first, on the
            // raw word (info bits 29-30 = 3; a compare the compiler does
            // not fold into a jump table with the other counts)
            // (the child count sits in bits 29-30 of the word, above the
            // first child's index: the compares need no shift)
            if (__builtin_expect(ent.x >= (3u << BH_NKIDS_SHIFT), 1))
                bh_group<4, COUNT, SC>(g, first, a, cn, stk, sp);
            else if (ent.x >= (2u << BH_NKIDS_SHIFT))
                bh_group<3, COUNT, SC>(g, first, a, cn, stk, sp);
            else if (ent.x >= (1u << BH_NKIDS_SHIFT))
                bh_group<2, COUNT, SC>(g, first, a, cn, stk, sp);
            else
                bh_group<1, COUNT, SC>(g, first, a, cn, stk, sp);
        } else {
            // children at depth D: all leaves, nothing to push
            if (ent.x >= (3u << BH_NKIDS_SHIFT))
                bh_group_leaves<4, COUNT, SC>(g, first, a, cn);
            else if (ent.x >= (2u << BH_NKIDS_SHIFT))
                bh_group_leaves<3, COUNT, SC>(g, first, a, cn);
            else if (ent.x >= (1u << BH_NKIDS_SHIFT))
                bh_group_leaves<2, COUNT, SC>(g, first, a, cn);
            else
                bh_group_leaves<1, COUNT, SC>(g, first, a, cn);
        }
        BH_DASSERT(sp <= CAP);  // the pushes stayed inside this warp's stack
        __syncwarp();
    }
    z = a.z;
    r0 = a.r0;
    r1 = a.r1;

    if (SC && valid) z -= 1.0;  // the self leaf's exact +1 (kScTheta)
    if (valid) {
        const int64_t o = slots ? slot
                                : (A.sorted_out ? t - t_begin : (int64_t)order[t]);
        A.rep[o] = make_float2((float)r0, (float)r1);
        if (A.zpart) A.zpart[o] = z;
        if (COUNT) A.counts[o] = make_int4(cn.internal, cn.leafnodes, cn.leafpts, cn.accepted);
    }
    // engine mode: Z from zpart[slot] by slot blocks (bh_step_zsum), the
    // same sums for any number of GPUs
    if (!slots)
        rep_z_tail(z, warp, lane, bid, nblk, s_z, &s_done, zblock, A.ticket,
                   A.z_out);
}

template <int D, bool COUNT, bool QUERY, bool SC>
__global__ void __launch_bounds__(kRepThreads, BH_REP_MIN_BLOCKS)
k_repulsive(const RepArgs A) {
    bh_pdl_trigger();  // the successor may launch early (PDL)
    bh_pdl_wait();     // the predecessor's results are visible

    rep_block<D, COUNT, QUERY, SC>(A, blockIdx.x, gridDim.x);
}
// Sum of gathered Z partials into *out (one CTA, cta_fold).
__global__ void __launch_bounds__(kFoldThreads)
k_fixed_sum(const double *__restrict__ x, int64_t n, double *__restrict__ out) {
    __shared__ double s_w[kFoldThreads / 32];
    const double s = cta_fold(x, n, s_w);
    if (threadIdx.x == 0) *out = s;
}

// ---------------------------------------------------------------------------
// Attractive CSR sweep: a group of G lanes per row; padded rows start at a
// multiple of 4 entries so each lane issues 128-bit loads of 4 column ids
// and 4 values (pad entries have value 0 and contribute exactly 0).
// ---------------------------------------------------------------------------
struct AttArgs {
    const int64_t *__restrict__ rp;
    const int32_t *__restrict__ col;
    const float *__restrict__ val;
    const float2 *__restrict__ y;
    int64_t row_begin, row_end;
    float exag_param;
    const bh_sched_t *__restrict__ sched;
    float2 *__restrict__ attr;
    // engine mode (part != NULL): the rows of att_rows (forces.cuh)
    const bh_part_t *__restrict__ part;
    int which;
};

// CTA `bid` of `nblk` sweeping CTAs of THREADS threads: row batches of
// THREADS / G rows, batch b handled by CTA b mod nblk.
template <int G, bool PADDED, int THREADS>
__device__ __forceinline__ void att_block(const AttArgs &A, int64_t bid,
                                          int64_t nblk) {
    static_assert(THREADS % G == 0, "whole row groups per CTA");
    constexpr int kRows = THREADS / G;
    const int64_t *__restrict__ rp = A.rp;
    const int32_t *__restrict__ col = A.col;
    const float *__restrict__ val = A.val;
    const float2 *__restrict__ y = A.y;
    int64_t row_begin, row_end;
    att_rows(A, row_begin, row_end);
    const bh_sched_t *__restrict__ sched = A.sched;
    const float exag = sched ? (sched->iteration < sched->exaggeration_iters
                                    ? sched->exaggeration
                                    : 1.0f)
                             : A.exag_param;
    const int gl = threadIdx.x % G;
    for (int64_t r0 = row_begin + bid * kRows; r0 < row_end;
         r0 += nblk * kRows) {
    const int64_t row = r0 + threadIdx.x / G;
    const bool ok = row < row_end;
    int64_t s = 0, e = 0;
    float2 yi = make_float2(0.f, 0.f);
    if (ok) {
        s = rp[row];
        e = rp[row + 1];
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
    if (PADDED) {
        // 32-bit offsets from the row start: fewer loop instructions than
        // 64-bit indices (a second loop body without the exaggeration
        // multiply made the fused kernel slower: code size)
        const int32_t *__restrict__ cp = col + s;
        const float *__restrict__ vp = val + s;
        const int len = (int)(e - s);
        for (int k = 4 * gl; k < len; k += 4 * G) {
            // the CSR stream bypasses L1 (no allocation) so that L1 holds the
            // y_j gathers
            const int4 c = ld_stream_i4(cp + k);
            const float4 v = ld_stream_f4(vp + k);
            const float2 y0 = __ldg(&y[c.x]), y1 = __ldg(&y[c.y]);
            const float2 y2 = __ldg(&y[c.z]), y3 = __ldg(&y[c.w]);
            float fx = 0.f, fy = 0.f;
            BH_ATTR_TERM(y0, v.x)
            BH_ATTR_TERM(y1, v.y)
            BH_ATTR_TERM(y2, v.z)
            BH_ATTR_TERM(y3, v.w)
            a0 += (double)fx;
            a1 += (double)fy;
        }
    } else {
        for (int64_t q = s + gl; q < e; q += G) {
            const int32_t c = col[q];
            const float v = val[q];
            const float2 yj = __ldg(&y[c]);
            float fx = 0.f, fy = 0.f;
            BH_ATTR_TERM(yj, v)
            a0 += (double)fx;
            a1 += (double)fy;
        }
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

#ifndef BH_ATTR_THREADS
#define BH_ATTR_THREADS 256
#endif
#ifndef BH_ATTR_MINB
#define BH_ATTR_MINB 8  // 32 registers: 0.518 ms vs 0.612 uncapped (C3 it. 600)
#endif
constexpr int kAttThreads = BH_ATTR_THREADS;

template <int G, bool PADDED>
__global__ void __launch_bounds__(kAttThreads, BH_ATTR_MINB)
k_attractive(const AttArgs A) {
    bh_pdl_trigger();  // the successor may launch early (PDL)
    bh_pdl_wait();     // the predecessor's results are visible

    att_block<G, PADDED, kAttThreads>(A, blockIdx.x, gridDim.x);
}

// ---------------------------------------------------------------------------
// Fused force pass: the traversal CTAs (issue-bound) and the CSR-sweep CTAs
// (L1/latency-bound) of one iteration in ONE grid, their block indices
// interleaved (na of every nr + na consecutive CTAs sweep) so that both kinds
// are co-resident on every SM and overlap, instead of running back to back.
// Each CTA computes exactly what it computes in its own kernel; the Z
// partials are indexed by traversal CTA, so Z is bitwise the same.
// ---------------------------------------------------------------------------
#ifndef BH_FORCES_MIN_BLOCKS
// 10 CTAs/SM for the fused pass (48 registers): its sweep CTAs gain more
// co-residency than the traversal CTAs lose (C3 iteration 600: 1.338 vs
// 1.450 ms at 9; the traversal alone prefers 9, BH_REP_MIN_BLOCKS)
#define BH_FORCES_MIN_BLOCKS 10
#endif
template <int D, int G, bool PADDED, bool SC>
__global__ void __launch_bounds__(kRepThreads, BH_FORCES_MIN_BLOCKS)
k_forces(const RepArgs R, const AttArgs A, int64_t nr, int64_t na) {
    bh_pdl_trigger();  // the successor may launch early (PDL)
    bh_pdl_wait();     // the predecessor's results are visible

    const int64_t b = blockIdx.x, nb = nr + na;
    const int64_t before = (b * na) / nb, upto = ((b + 1) * na) / nb;
    if (upto > before)
        att_block<G, PADDED, kRepThreads>(A, before, na);
    else
        rep_block<D, false, false, SC>(R, b - upto, nr);
}

// ---------------------------------------------------------------------------
// Exact O(N^2) repulsion (forces.py:153-173): the end-of-run KL needs the
// exact Z.  Tiles of points staged in shared memory; f32 pair math, f32
// partial per tile, f64 accumulation.
// ---------------------------------------------------------------------------
constexpr int kExTile = 1024;

__global__ void __launch_bounds__(256)
k_repulsive_exact(const float2 *__restrict__ y, int64_t n,
                  float2 *__restrict__ rep, double *__restrict__ zpart,
                  double *__restrict__ zblock, unsigned *__restrict__ ticket,
                  double *__restrict__ z_out) {
    __shared__ float2 s_y[kExTile];
    __shared__ double s_z[8];
    __shared__ bool s_last;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool ok = i < n;
    const float2 yi = ok ? y[i] : make_float2(0.f, 0.f);
    double z = 0.0, r0 = 0.0, r1 = 0.0;
    for (int64_t j0 = 0; j0 < n; j0 += kExTile) {
        __syncthreads();
        for (int q = threadIdx.x; q < kExTile; q += blockDim.x)
            s_y[q] = j0 + q < n ? y[j0 + q] : make_float2(0.f, 0.f);
        __syncthreads();
        const int nb = (n - j0) < kExTile ? (int)(n - j0) : kExTile;
        // (the same pair arithmetic as the traversal: rcp.approx, FMA)
        const int qself = (i >= j0 && i < j0 + kExTile) ? (int)(i - j0) : -1;
        float fz = 0.f, fx = 0.f, fy = 0.f;
#pragma unroll 4
        for (int q = 0; q < nb; q++) {
            const float2 p = s_y[q];
            const float dx = yi.x - p.x, dy = yi.y - p.y;
            float k = rcp_approx(1.0f + fmaf(dx, dx, dy * dy));
            k = q == qself ? 0.f : k;
            const float k2 = k * k;
            fz += k;
            fx = fmaf(k2, dx, fx);
            fy = fmaf(k2, dy, fy);
        }
        z += (double)fz;
        r0 += (double)fx;
        r1 += (double)fy;
    }
    if (ok) {
        if (rep) rep[i] = make_float2((float)r0, (float)r1);
        if (zpart) zpart[i] = z;
    }
    double wz = warp_sum(ok ? z : 0.0);
    if ((threadIdx.x & 31) == 0) s_z[threadIdx.x >> 5] = wz;
    __syncthreads();
    if (threadIdx.x == 0) {
        double bz = 0.0;
        for (int w = 0; w < 8; w++) bz += s_z[w];
        zblock[blockIdx.x] = bz;
        __threadfence();
        s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        __threadfence();
        double tot = 0.0;
        for (unsigned b = 0; b < gridDim.x; b++) tot += __ldcg(&zblock[b]);
        *z_out = tot;
        *ticket = 0;
    }
}

// KL rows (optimizer.py:227-239) in f64, one warp per row.
template <typename T>
__global__ void __launch_bounds__(256)
k_kl_rows(const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
          const T *__restrict__ val, int64_t n, const p2_t<T> *__restrict__ y,
          const double *__restrict__ zp, double *__restrict__ part,
          unsigned *__restrict__ ticket, double *__restrict__ kl_out) {
    __shared__ double s_a[8];
    __shared__ bool s_last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double Z = *zp;
    double acc = 0.0;
    for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < n;
         row += (int64_t)gridDim.x * 8) {
        const p2_t<T> yi = y[row];
        for (int64_t q = rp[row] + lane; q < rp[row + 1]; q += 32) {
            const T p = val[q];
            if (p == T(0)) continue;  // padding
            const p2_t<T> yj = y[col[q]];
            double dx = (double)yi.x - (double)yj.x;
            double dy = (double)yi.y - (double)yj.y;
            double pd = (double)p;
            acc += pd * log(pd * Z * (1.0 + dx * dx + dy * dy));
        }
    }
    acc = warp_sum(acc);
    if (lane == 0) s_a[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int w = 0; w < 8; w++) b += s_a[w];
        part[blockIdx.x] = b;
        __threadfence();
        s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        __threadfence();
        double tot = 0.0;
        for (unsigned b = 0; b < gridDim.x; b++) tot += __ldcg(&part[b]);
        *kl_out = tot;
        *ticket = 0;
    }
}


}  // namespace bh

using namespace bh;

extern "C" size_t bh_repulsive_workspace_bytes(int64_t n) {
    return bh_align(sizeof(double) * rep_grid(n)) + 256;
}

extern "C" int bh_repulsive(const bh_tree_t *t, const bh_bounds_t *bounds,
                            double theta, const float *y_query,
                            int64_t t_begin, int64_t t_end, int sorted_out,
                            float *rep, double *zpart, double *zblock,
                            double *z_out, int32_t *counts, void *ws,
                            size_t ws_bytes, bh_stream_t stream) {
    BH_REQUIRE(theta >= 0, "theta must be >= 0, got %g", theta);
    BH_REQUIRE(t->precision != 64, "precision-64 tree: use the _f64 entry point");
    BH_REQUIRE(t_begin >= 0 && t_end <= t->n_points && t_begin <= t_end,
               "bad point range");
    if (t_end == t_begin) return BH_OK;
    const int grid = rep_grid(t_end - t_begin);
    BH_REQUIRE(ws_bytes >= bh_repulsive_workspace_bytes(t_end - t_begin),
               "repulsive workspace too small");
    char *w = (char *)ws;
    if (!zblock) zblock = (double *)w;
    unsigned *ticket = (unsigned *)(w + bh_align(sizeof(double) * grid));
    cudaStream_t st = bh_cs(stream);
    const RepArgs A{(const float4 *)t->node, (const float2 *)t->ys, t->order,
                    (const float2 *)y_query, bounds, t->status, theta, t_begin,
                    t_end, sorted_out, (float2 *)rep, zpart, (int4 *)counts,
                    zblock, ticket, z_out};
    const bool sc = theta <= kScTheta;
#define BH_REP_LAUNCH(D, CNT, Q, SC)                                          \
    BH_LAUNCH("k_repulsive", (k_repulsive<D, CNT, Q, SC>), grid, kRepThreads, 0, st, A)
#define BH_REP_LAUNCH2(D)                                                     \
    if (y_query) {                                                            \
        if (counts) BH_REP_LAUNCH(D, true, true, false);                      \
        else BH_REP_LAUNCH(D, false, true, false);                            \
    } else if (sc) {                                                          \
        if (counts) BH_REP_LAUNCH(D, true, false, true);                      \
        else BH_REP_LAUNCH(D, false, false, true);                            \
    } else {                                                                  \
        if (counts) BH_REP_LAUNCH(D, true, false, false);                     \
        else BH_REP_LAUNCH(D, false, false, false);                           \
    }
    if (t->code_bits == 32) {
        BH_REP_LAUNCH2(16)
    } else if (t->code_bits == 64) {
        BH_REP_LAUNCH2(32)
    } else {
        return set_error(BH_ERR_UNSUPPORTED, "code_bits must be 32 or 64");
    }
#undef BH_REP_LAUNCH
#undef BH_REP_LAUNCH2
    BH_CHECK_LAUNCH("k_repulsive");
    return BH_OK;
}

extern "C" int bh_sum_partials(const double *x, int64_t n, double *out,
                               bh_stream_t stream) {
    k_fixed_sum<<<1, kFoldThreads, 0, bh_cs(stream)>>>(x, n, out);
    BH_CHECK_LAUNCH("k_fixed_sum");
    return BH_OK;
}

extern "C" int bh_attractive(const int64_t *row_ptr, const int32_t *col,
                             const float *val, int64_t n_rows, int padded,
                             const float *y, int64_t row_begin,
                             int64_t row_end, float exaggeration,
                             const bh_sched_t *sched, float *attr,
                             bh_stream_t stream) {
    BH_REQUIRE(row_begin >= 0 && row_end <= n_rows && row_begin <= row_end,
               "bad row range");
    if (row_end == row_begin) return BH_OK;
    // lanes per row (tuning knob BH_ATTR_G; default 16, measured best at C3:
    // tools/microbench.py, profiles/r01_microbench.txt)
    static const int g_env = [] {
        const char *s = getenv("BH_ATTR_G");
        int g = s ? atoi(s) : 16;
        return (g == 4 || g == 8 || g == 16 || g == 32) ? g : 16;
    }();
    cudaStream_t st = bh_cs(stream);
    const AttArgs A{row_ptr, col, val, (const float2 *)y, row_begin, row_end,
                    exaggeration, sched, (float2 *)attr};
#define BH_ATTR(G)                                                            \
    {                                                                         \
        const int grid = bh_blocks(row_end - row_begin, kAttThreads / G);     \
        if (padded)                                                           \
            BH_LAUNCH("k_attractive", (k_attractive<G, true>), grid,          \
                      kAttThreads, 0, st, A);                                 \
        else                                                                  \
            BH_LAUNCH("k_attractive", (k_attractive<G, false>), grid,         \
                      kAttThreads, 0, st, A);                                 \
    }
    switch (g_env) {
        case 4: BH_ATTR(4) break;
        case 8: BH_ATTR(8) break;
        case 32: BH_ATTR(32) break;
        default: BH_ATTR(16) break;
    }
#undef BH_ATTR
    BH_CHECK_LAUNCH("k_attractive");
    return BH_OK;
}

extern "C" int bh_forces(const bh_tree_t *t, const bh_bounds_t *bounds,
                         double theta, int64_t t_begin, int64_t t_end,
                         int sorted_out, float *rep, double *zblock,
                         double *z_out, void *ws, size_t ws_bytes,
                         const int64_t *row_ptr, const int32_t *col,
                         const float *val, int64_t n_rows, int padded,
                         const float *y, int64_t row_begin, int64_t row_end,
                         float exaggeration, const bh_sched_t *sched,
                         float *attr, bh_stream_t stream) {
    BH_REQUIRE(theta >= 0, "theta must be >= 0, got %g", theta);
    BH_REQUIRE(t->precision != 64, "precision-64 tree: use the _f64 entry point");
    BH_REQUIRE(t_begin >= 0 && t_end <= t->n_points && t_begin <= t_end,
               "bad point range");
    BH_REQUIRE(row_begin >= 0 && row_end <= n_rows && row_begin <= row_end,
               "bad row range");
    if (t_end == t_begin || row_end == row_begin) {
        // nothing to overlap: the separate kernels
        int rc = bh_attractive(row_ptr, col, val, n_rows, padded, y, row_begin,
                               row_end, exaggeration, sched, attr, stream);
        if (rc != BH_OK) return rc;
        return bh_repulsive(t, bounds, theta, nullptr, t_begin, t_end,
                            sorted_out, rep, nullptr, zblock, z_out, nullptr,
                            ws, ws_bytes, stream);
    }
    BH_REQUIRE(ws_bytes >= bh_repulsive_workspace_bytes(t_end - t_begin),
               "repulsive workspace too small");
    // sweeping CTAs per traversal CTA (tuning knob BH_FUSE_RATIO = nr / na)
    static const double ratio = [] {
        const char *s = getenv("BH_FUSE_RATIO");
        const double r = s ? atof(s) : 2.0;
        return r > 0.0 ? r : 2.0;
    }();
#ifndef BH_FUSE_G
#define BH_FUSE_G 16
#endif
    constexpr int G = BH_FUSE_G;
    const int64_t nr = rep_grid(t_end - t_begin);
    const int64_t na = std::max<int64_t>(
        1, std::min<int64_t>((int64_t)ceil((double)nr / ratio),
                             bh_blocks(row_end - row_begin, kRepThreads / G)));
    char *w = (char *)ws;
    if (!zblock) zblock = (double *)w;
    unsigned *ticket = (unsigned *)(w + bh_align(sizeof(double) * nr));
    const RepArgs R{(const float4 *)t->node, (const float2 *)t->ys, t->order,
                    nullptr, bounds, t->status, theta, t_begin, t_end,
                    sorted_out, (float2 *)rep, nullptr, nullptr, zblock, ticket,
                    z_out};
    const AttArgs A{row_ptr, col, val, (const float2 *)y, row_begin, row_end,
                    exaggeration, sched, (float2 *)attr};
    cudaStream_t st = bh_cs(stream);
    const unsigned grid = (unsigned)(nr + na);
#define BH_FORCES1(D, SC)                                                     \
    if (padded)                                                               \
        BH_LAUNCH("k_forces", (k_forces<D, G, true, SC>), grid, kRepThreads,  \
                  0, st, R, A, nr, na);                                       \
    else                                                                      \
        BH_LAUNCH("k_forces", (k_forces<D, G, false, SC>), grid, kRepThreads, \
                  0, st, R, A, nr, na);
#define BH_FORCES(D)                                                          \
    if (theta <= kScTheta) {                                                  \
        BH_FORCES1(D, true)                                                   \
    } else {                                                                  \
        BH_FORCES1(D, false)                                                  \
    }
    if (t->code_bits == 32) {
        BH_FORCES(16)
    } else if (t->code_bits == 64) {
        BH_FORCES(32)
    } else {
        return set_error(BH_ERR_UNSUPPORTED, "code_bits must be 32 or 64");
    }
#undef BH_FORCES
#undef BH_FORCES1
    BH_CHECK_LAUNCH("k_forces");
    return BH_OK;
}

extern "C" size_t bh_repulsive_exact_workspace_bytes(int64_t n) {
    return bh_align(sizeof(double) * bh_blocks(n, 256)) + 256;
}

extern "C" int bh_repulsive_exact(const float *y, int64_t n, float *rep,
                                  double *zpart, double *z_out, void *ws,
                                  size_t ws_bytes, bh_stream_t stream) {
    BH_REQUIRE(n >= 2, "need at least 2 points");
    BH_REQUIRE(ws_bytes >= bh_repulsive_exact_workspace_bytes(n),
               "exact workspace too small");
    const int grid = bh_blocks(n, 256);
    char *w = (char *)ws;
    k_repulsive_exact<<<grid, 256, 0, bh_cs(stream)>>>(
        (const float2 *)y, n, (float2 *)rep, zpart, (double *)w,
        (unsigned *)(w + bh_align(sizeof(double) * grid)), z_out);
    BH_CHECK_LAUNCH("k_repulsive_exact");
    return BH_OK;
}

extern "C" size_t bh_kl_workspace_bytes(int64_t n) {
    return bh_align(sizeof(double) * kSMs * 8) + 256;
}

template <typename T>
static int kl_impl(const int64_t *row_ptr, const int32_t *col, const T *val,
                   int64_t n, const T *y, const double *z, double *kl_out,
                   void *ws, size_t ws_bytes, bh_stream_t stream) {
    // pad entries carry p == 0 and are skipped
    BH_REQUIRE(ws_bytes >= bh_kl_workspace_bytes(n), "kl workspace too small");
    int grid = bh_blocks(n, 8);
    if (grid > kSMs * 8) grid = kSMs * 8;
    char *w = (char *)ws;
    k_kl_rows<T><<<grid, 256, 0, bh_cs(stream)>>>(
        row_ptr, col, val, n, (const p2_t<T> *)y, z, (double *)w,
        (unsigned *)(w + bh_align(sizeof(double) * kSMs * 8)), kl_out);
    BH_CHECK_LAUNCH("k_kl_rows");
    return BH_OK;
}

extern "C" int bh_kl_rows(const int64_t *row_ptr, const int32_t *col,
                          const float *val, int64_t n, int padded,
                          const float *y, const double *z, double *kl_out,
                          void *ws, size_t ws_bytes, bh_stream_t stream) {
    (void)padded;
    return kl_impl(row_ptr, col, val, n, y, z, kl_out, ws, ws_bytes, stream);
}

extern "C" int bh_kl_rows_f64(const int64_t *row_ptr, const int32_t *col,
                              const double *val, int64_t n, int padded,
                              const double *y, const double *z, double *kl_out,
                              void *ws, size_t ws_bytes, bh_stream_t stream) {
    (void)padded;
    return kl_impl(row_ptr, col, val, n, y, z, kl_out, ws, ws_bytes, stream);
}

// ---------------------------------------------------------------------------
// Engine entry points (the share of bh_part_t; storage-slot traversal).
// ---------------------------------------------------------------------------
namespace bh {
static int fuse_na(int64_t nr, int64_t rows, int rows_per_cta) {
    static const double ratio = [] {
        const char *s = getenv("BH_FUSE_RATIO");
        const double r = s ? atof(s) : 2.0;
        return r > 0.0 ? r : 2.0;
    }();
    return (int)std::max<int64_t>(
        1, std::min<int64_t>((int64_t)ceil((double)nr / ratio),
                             bh_blocks(rows, rows_per_cta)));
}
}  // namespace bh

extern "C" int bh_step_attractive(const int64_t *row_ptr, const int32_t *col,
                                  const float *val, int padded, const float *y,
                                  const bh_part_t *part, int64_t max_rows,
                                  const bh_sched_t *sched, float *attr,
                                  bh_stream_t stream) {
    BH_REQUIRE(part && sched, "part and sched are required");
    if (max_rows <= 0) return BH_OK;
    constexpr int G = 16;
    const AttArgs A{row_ptr, col, val, (const float2 *)y, 0, 0, 1.0f, sched,
                    (float2 *)attr, part, 0};
    const int grid = bh_blocks(max_rows, kAttThreads / G);
    if (padded)
        BH_LAUNCH("k_attractive", (k_attractive<G, true>), grid, kAttThreads,
                  0, bh_cs(stream), A);
    else
        BH_LAUNCH("k_attractive", (k_attractive<G, false>), grid, kAttThreads,
                  0, bh_cs(stream), A);
    BH_CHECK_LAUNCH("k_attractive");
    return BH_OK;
}

extern "C" int bh_step_forces(const bh_tree_t *t, const bh_bounds_t *bounds,
                              double theta, const float *y,
                              const int32_t *rank, const int32_t *qlist,
                              const bh_part_t *part, int64_t max_points,
                              int mode, float *rep, double *zpart, void *ws,
                              size_t ws_bytes, const int64_t *row_ptr,
                              const int32_t *col, const float *val,
                              int padded, const bh_sched_t *sched,
                              float *attr, bh_stream_t stream) {
    BH_REQUIRE(theta >= 0, "theta must be >= 0, got %g", theta);
    BH_REQUIRE(t->precision != 64, "precision-64 tree: use the _f64 entry point");
    BH_REQUIRE(part && y && rank && zpart && sched,
               "part, y, rank, zpart and sched are required");
    BH_REQUIRE(mode >= 0 && mode <= 2, "mode must be 0 (fused), 1 or 2");
    BH_REQUIRE(max_points >= 1 && max_points <= t->n_points,
               "bad max_points");
    BH_REQUIRE(ws_bytes >= bh_repulsive_workspace_bytes(max_points),
               "repulsive workspace too small");
    constexpr int G = 16;
    const int64_t nr = rep_grid(max_points);
    unsigned *ticket = (unsigned *)((char *)ws + bh_align(sizeof(double) * nr));
    const RepArgs R{(const float4 *)t->node, (const float2 *)t->ys, t->order,
                    (const float2 *)y, bounds, t->status, theta, 0,
                    t->n_points, 0, (float2 *)rep, zpart, nullptr, nullptr,
                    ticket, nullptr, part, rank, qlist};
    const AttArgs A{row_ptr, col, val, (const float2 *)y, 0, 0, 1.0f, sched,
                    (float2 *)attr, part, 1};
    const bool sc = theta <= kScTheta;
    cudaStream_t st = bh_cs(stream);
    if (mode == 2) {  // the sweep of rows [split, hi) alone
        const int grid = bh_blocks(max_points, kAttThreads / G);
        if (padded)
            BH_LAUNCH("k_attractive", (k_attractive<G, true>), grid,
                      kAttThreads, 0, st, A);
        else
            BH_LAUNCH("k_attractive", (k_attractive<G, false>), grid,
                      kAttThreads, 0, st, A);
        BH_CHECK_LAUNCH("k_attractive");
        return BH_OK;
    }
#define BH_STEP_REP(D, SC)                                                    \
    BH_LAUNCH("k_repulsive", (k_repulsive<D, false, false, SC>), (int)nr,     \
              kRepThreads, 0, st, R)
#define BH_STEP_FUSED(D, SC)                                                  \
    {                                                                         \
        const int64_t na = fuse_na(nr, max_points, kRepThreads / G);          \
        if (padded)                                                           \
            BH_LAUNCH("k_forces", (k_forces<D, G, true, SC>),                 \
                      (unsigned)(nr + na), kRepThreads, 0, st, R, A, nr, na); \
        else                                                                  \
            BH_LAUNCH("k_forces", (k_forces<D, G, false, SC>),                \
                      (unsigned)(nr + na), kRepThreads, 0, st, R, A, nr, na); \
    }
#define BH_STEP(D)                                                            \
    if (mode == 1) {                                                          \
        if (sc) BH_STEP_REP(D, true); else BH_STEP_REP(D, false);             \
    } else {                                                                  \
        if (sc) BH_STEP_FUSED(D, true) else BH_STEP_FUSED(D, false)           \
    }
    if (t->code_bits == 32) {
        BH_STEP(16)
    } else if (t->code_bits == 64) {
        BH_STEP(32)
    } else {
        return set_error(BH_ERR_UNSUPPORTED, "code_bits must be 32 or 64");
    }
#undef BH_STEP
#undef BH_STEP_FUSED
#undef BH_STEP_REP
    BH_CHECK_LAUNCH("k_forces");
    return BH_OK;
}
