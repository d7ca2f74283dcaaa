// Force kernels of the f64 run mode (the reference's default precision,
// io.py:21-30): float64 coordinates, values and forces, and every pair term
// in float64 with the reference's operation order and no FMA contraction
// (forces.py:56-82, 85-150, 153-182):
//   attractive  pq = v / ((1 + dx*dx) + dy*dy);   a += pq * dx
//   leaf point  k = 1 / ((1 + dx*dx) + dy*dy);   z += k;  r += (k*k) * dx
//   cell        d2 = dx*dx + dy*dy;  accept iff side*side < theta^2 * d2;
//               k = 1 / (1 + d2);  mk = m * k;  z += mk;  r += (mk*k) * dx
// The traversal is the f32 path's warp-synchronous walk (forces.cu) with the
// acceptance test in the reference's own f64 form: a stack entry carries
// side^2 of the children's cells (exact quartering per level) instead of
// side^2 / theta^2.
#include <algorithm>

#include "forces.cuh"

namespace bh {

using Rec64 = NodeRec<double>;

__device__ __forceinline__ void leaf_pair64(double2 yi, double2 p, Acc64 &a) {
    const double dx = __dsub_rn(yi.x, p.x), dy = __dsub_rn(yi.y, p.y);
    const double k = __drcp_rn(__dadd_rn(__dadd_rn(1.0, __dmul_rn(dx, dx)),
                                             __dmul_rn(dy, dy)));
    a.z = __dadd_rn(a.z, k);
    const double k2 = __dmul_rn(k, k);
    a.r0 = __dadd_rn(a.r0, __dmul_rn(k2, dx));
    a.r1 = __dadd_rn(a.r1, __dmul_rn(k2, dy));
}

struct Ctx64 {
    const void *__restrict__ node;
    const double2 *__restrict__ ys;
    double2 yi;
    double side2, theta2;
    bool mine;
    uint32_t self;
    int lane;
};

// One child for one lane; returns the ballot of lanes that open it.
template <bool COUNT>
__device__ __forceinline__ uint32_t bh_child64(const Ctx64 &g, double2 c,
                                               uint32_t m, uint32_t info,
                                               Acc64 &a, RepCounts &cn) {
    if (info & BH_LEAF_BIT) {  // warp-uniform
        const uint32_t s = info & ~BH_LEAF_BIT;
        if (COUNT && g.mine) {
            cn.leafnodes++;
            cn.leafpts += (int)m;
        }
        if (m == 1u) {
            if (g.mine && s != g.self) leaf_pair64(g.yi, c, a);
            return 0;
        }
        // coincident-code bucket: the points in order, loaded once per 32
        for (uint32_t b = 0; b < m; b += 32) {
            const double2 pq = (b + g.lane < m) ? g.ys[s + b + g.lane]
                                                : make_double2(0.0, 0.0);
            const int nb = (int)min(32u, m - b);
            for (int jj = 0; jj < nb; jj++) {
                const double2 p = make_double2(__shfl_sync(0xffffffffu, pq.x, jj),
                                               __shfl_sync(0xffffffffu, pq.y, jj));
                if (g.mine && s + b + jj != g.self) leaf_pair64(g.yi, p, a);
            }
        }
        return 0;
    }
    const double dx = __dsub_rn(g.yi.x, c.x), dy = __dsub_rn(g.yi.y, c.y);
    const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
    const bool acc = g.side2 < __dmul_rn(g.theta2, d2);
    if (COUNT && g.mine) {
        cn.internal++;
        cn.accepted += acc;
    }
    if (g.mine && acc) {
        const double k = __drcp_rn(__dadd_rn(1.0, d2));
        const double mk = __dmul_rn((double)m, k);
        a.z = __dadd_rn(a.z, mk);
        const double mk2 = __dmul_rn(mk, k);
        a.r0 = __dadd_rn(a.r0, __dmul_rn(mk2, dx));
        a.r1 = __dadd_rn(a.r1, __dmul_rn(mk2, dy));
    }
    // lanes outside the mask carry side2 = -1 (Ctx64): they accept every
    // cell, so the ballot of the lanes that open it needs no mask term
    return ballot_full(!acc);
}

// The CNT children of one popped group, in order (the reference's
// accumulation order); lane c keeps child c's info word and push mask.
template <int CNT, bool COUNT>
__device__ __forceinline__ void group64(const Ctx64 &g, const void *node,
                                        uint32_t first, Acc64 &a,
                                        RepCounts &cn, uint32_t &info,
                                        uint32_t &msk) {
    double2 cc[CNT];
    uint2 mi[CNT];
#pragma unroll
    for (int c = 0; c < CNT; c++) {
        cc[c] = __ldg((const double2 *)node + 2 * (first + c));
        mi[c] = __ldg((const uint2 *)node + 4 * (first + c) + 2);
    }
#pragma unroll
    for (int c = 0; c < CNT; c++) {
        const uint32_t need = bh_child64<COUNT>(g, cc[c], mi[c].x, mi[c].y, a, cn);
        if (g.lane == c) {
            info = mi[c].y;
            msk = need;
        }
    }
}

struct RepArgs64 {
    const void *__restrict__ node;
    const double2 *__restrict__ ys;
    const int32_t *__restrict__ order;
    const double2 *__restrict__ y_query;
    const bh_bounds_t *__restrict__ bounds;
    const int32_t *__restrict__ status;
    double theta;
    int64_t t_begin, t_end;
    int sorted_out;
    double2 *__restrict__ rep;
    double *__restrict__ zpart;
    int4 *__restrict__ counts;
    double *__restrict__ zblock;
    unsigned *__restrict__ ticket;
    double *__restrict__ z_out;
    const bh_part_t *__restrict__ part;  // engine mode (forces.cu RepArgs)
    const int32_t *__restrict__ rank;
    const int32_t *__restrict__ qlist;
};

__device__ __forceinline__ uint4 side2_entry(uint32_t info, uint32_t msk,
                                             double side2) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(side2);
    return make_uint4(info, msk, (uint32_t)b, (uint32_t)(b >> 32));
}

// Traversal CTA `bid` of `nblk`: sorted positions t_begin + 128 bid + [0, 128).
template <int D, bool COUNT, bool QUERY>
__device__ __forceinline__ void rep_block64(const RepArgs64 &A, int64_t bid,
                                            int64_t nblk) {
    constexpr int CAP = 3 * D + 2;
    __shared__ uint4 s_stack[kRepWarps][CAP];
    __shared__ double s_z[kRepWarps];
    __shared__ unsigned s_done;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool slots = A.part != nullptr;
    const int64_t lo = slots ? 0 : A.t_begin;
    const int64_t hi = slots ? A.part->hi - A.part->lo : A.t_end;
    if (lo + bid * kRepThreads >= hi) return;  // engine mode: past the share
    if (threadIdx.x == 0) s_done = 0;
    __syncthreads();
    const int64_t t = lo + (bid * kRepWarps + warp) * 32 + lane;
    const bool valid = t < hi && *A.status == BH_OK;
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    double2 yi = make_double2(0.0, 0.0);
    uint32_t self = (uint32_t)t;
    int64_t slot = 0;
    if (valid) {
        if (slots && A.qlist) {
            slot = A.qlist[t];
            yi = A.y_query[slot];
            self = (uint32_t)A.rank[slot];
        } else if (slots) {
            slot = A.order[t];
            yi = A.ys[t];
        } else {
            yi = QUERY ? A.y_query[A.order[t]] : A.ys[t];
        }
    }
    const double theta2 = __dmul_rn(A.theta, A.theta);
    Acc64 a{0.0, 0.0, 0.0};
    RepCounts cn = {0, 0, 0, 0};
    uint4 *stk = s_stack[warp];
    int sp = 0;
    if (act) {
        if (lane == 0) {
            // the root "group": node 0 alone, side = 2 r_span
            const double side = __dmul_rn(2.0, A.bounds->r_span);
            stk[0] = side2_entry(0u, act, __dmul_rn(side, side));
        }
        sp = 1;
        __syncwarp();
    }
    while (sp > 0) {
        // (no barrier after the read: the ballots below depend on `ent` in
        // every lane; the barrier at the end orders the pushes)
        const uint4 ent = stk[--sp];
        const uint32_t first = ent.x & BH_CHILD_MASK;
        const int cnt = (int)(ent.x >> BH_NKIDS_SHIFT) + 1;
        const double side2 = __longlong_as_double(
            (long long)(((unsigned long long)ent.w << 32) | ent.z));
        const bool mine = ((ent.y >> lane) & 1u) != 0;
        const Ctx64 g{A.node, A.ys, yi, mine ? side2 : -1.0, theta2, mine, self,
                      lane};
        uint32_t info = 0, msk = 0;
        // straight-line code per (warp-uniform) child count, every record of
        // the group loaded up front; full groups tested first on the raw word
        if (ent.x >= (3u << BH_NKIDS_SHIFT))
            group64<4, COUNT>(g, A.node, first, a, cn, info, msk);
        else if (cnt == 3)
            group64<3, COUNT>(g, A.node, first, a, cn, info, msk);
        else if (cnt == 2)
            group64<2, COUNT>(g, A.node, first, a, cn, info, msk);
        else
            group64<1, COUNT>(g, A.node, first, a, cn, info, msk);
        // lane c pushes child c's group if any lane opens it; one ballot
        // gives every writer its slot (child 0 ends on top)
        const bool push = msk != 0u;
        const uint32_t nz = ballot_full(push);
        if (push)
            stk[sp + __popc(nz >> (lane + 1))] =
                side2_entry(info, msk, __dmul_rn(side2, 0.25));
        sp += __popc(nz);
        __syncwarp();
    }
    if (valid) {
        const int64_t o = slots ? slot
                                : (A.sorted_out ? t - A.t_begin : (int64_t)A.order[t]);
        A.rep[o] = make_double2(a.r0, a.r1);
        if (A.zpart) A.zpart[o] = a.z;
        if (COUNT) A.counts[o] = make_int4(cn.internal, cn.leafnodes, cn.leafpts, cn.accepted);
    }
    if (!slots)  // engine mode: bh_step_zsum
        rep_z_tail(a.z, warp, lane, bid, nblk, s_z, &s_done, A.zblock,
                   A.ticket, A.z_out);
}

template <int D, bool COUNT, bool QUERY>
__global__ void __launch_bounds__(kRepThreads)
k_repulsive64(const RepArgs64 A) {
    bh_pdl_trigger();
    bh_pdl_wait();
    rep_block64<D, COUNT, QUERY>(A, blockIdx.x, gridDim.x);
}

struct AttArgs64 {
    const int64_t *__restrict__ rp;
    const int32_t *__restrict__ col;
    const double *__restrict__ val;
    const double2 *__restrict__ y;
    int64_t row_begin, row_end;
    double exag_param;
    const bh_sched_t *__restrict__ sched;
    double2 *__restrict__ attr;
    const bh_part_t *__restrict__ part;  // engine mode (att_rows, forces.cuh)
    int which;
};

// Attractive sweep CTA `bid` of `nblk` (THREADS threads), G lanes per row
// (forces.py:56-71 in f64).
template <int G, bool PADDED, int THREADS>
__device__ __forceinline__ void att_block64(const AttArgs64 &A, int64_t bid,
                                            int64_t nblk) {
    constexpr int kRows = THREADS / G;
    const int64_t *__restrict__ rp = A.rp;
    const int32_t *__restrict__ col = A.col;
    const double *__restrict__ val = A.val;
    const double2 *__restrict__ y = A.y;
    int64_t row_begin, row_end;
    att_rows(A, row_begin, row_end);
    const bh_sched_t *__restrict__ sched = A.sched;
    const double exag = sched ? (sched->iteration < sched->exaggeration_iters
                                     ? sched->exaggeration_f64
                                     : 1.0)
                              : A.exag_param;
    const int gl = threadIdx.x % G;
    for (int64_t r0 = row_begin + bid * kRows; r0 < row_end;
         r0 += nblk * kRows) {
        const int64_t row = r0 + threadIdx.x / G;
        const bool ok = row < row_end;
        int64_t s = 0, e = 0;
        double2 yi = make_double2(0.0, 0.0);
        if (ok) {
            s = rp[row];
            e = rp[row + 1];
            yi = y[row];
        }
        double a0 = 0.0, a1 = 0.0;
        auto term = [&](const double2 yj, double v) {
            const double dx = __dsub_rn(yi.x, yj.x), dy = __dsub_rn(yi.y, yj.y);
            const double pq = __ddiv_rn(
                __dmul_rn(v, exag),
                __dadd_rn(__dadd_rn(1.0, __dmul_rn(dx, dx)), __dmul_rn(dy, dy)));
            a0 = __dadd_rn(a0, __dmul_rn(pq, dx));
            a1 = __dadd_rn(a1, __dmul_rn(pq, dy));
        };
        if (PADDED) {
            for (int64_t q = s + 4 * gl; q < e; q += 4 * G) {
                const int4 c = ld_stream_i4(col + q);
                const double2 v01 = ld_stream_d2(val + q);
                const double2 v23 = ld_stream_d2(val + q + 2);
                // all four gathers in flight before the arithmetic
                const double2 y0 = __ldg(&y[c.x]), y1 = __ldg(&y[c.y]);
                const double2 y2 = __ldg(&y[c.z]), y3 = __ldg(&y[c.w]);
                term(y0, v01.x);
                term(y1, v01.y);
                term(y2, v23.x);
                term(y3, v23.y);
            }
        } else {
            for (int64_t q = s + gl; q < e; q += G) term(__ldg(&y[col[q]]), val[q]);
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            a0 = __dadd_rn(a0, __shfl_xor_sync(0xffffffffu, a0, o));
            a1 = __dadd_rn(a1, __shfl_xor_sync(0xffffffffu, a1, o));
        }
        if (ok && gl == 0) A.attr[row] = make_double2(a0, a1);
    }
}

template <int G, bool PADDED>
__global__ void __launch_bounds__(256) k_attractive64(const AttArgs64 A) {
    bh_pdl_trigger();
    bh_pdl_wait();
    att_block64<G, PADDED, 256>(A, blockIdx.x, gridDim.x);
}

// The fused f64 force pass (the f32 k_forces, forces.cu): traversal and sweep
// CTAs interleaved nr : na by block index.
template <int D, int G, bool PADDED>
__global__ void __launch_bounds__(kRepThreads)
k_forces64(const RepArgs64 R, const AttArgs64 A, int64_t nr, int64_t na) {
    bh_pdl_trigger();
    bh_pdl_wait();
    const int64_t b = blockIdx.x, nb = nr + na;
    const int64_t before = (b * na) / nb, upto = ((b + 1) * na) / nb;
    if (upto > before)
        att_block64<G, PADDED, kRepThreads>(A, before, na);
    else
        rep_block64<D, false, false>(R, b - upto, nr);
}

// Exact O(N^2) repulsion in f64 (forces.py:153-173), tiles in shared memory.
constexpr int kExTile64 = 512;

__global__ void __launch_bounds__(256)
k_repulsive_exact64(const double2 *__restrict__ y, int64_t n,
                    double2 *__restrict__ rep, double *__restrict__ zpart,
                    double *__restrict__ zblock, unsigned *__restrict__ ticket,
                    double *__restrict__ z_out) {
    __shared__ double2 s_y[kExTile64];
    __shared__ double s_z[8];
    __shared__ bool s_last;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool ok = i < n;
    const double2 yi = ok ? y[i] : make_double2(0.0, 0.0);
    Acc64 a{0.0, 0.0, 0.0};
    for (int64_t j0 = 0; j0 < n; j0 += kExTile64) {
        __syncthreads();
        for (int q = threadIdx.x; q < kExTile64; q += blockDim.x)
            s_y[q] = j0 + q < n ? y[j0 + q] : make_double2(0.0, 0.0);
        __syncthreads();
        const int nb = (n - j0) < kExTile64 ? (int)(n - j0) : kExTile64;
        for (int q = 0; q < nb; q++)
            if (j0 + q != i) leaf_pair64(yi, s_y[q], a);
    }
    if (ok) {
        if (rep) rep[i] = make_double2(a.r0, a.r1);
        if (zpart) zpart[i] = a.z;
    }
    double wz = warp_sum(ok ? a.z : 0.0);
    if ((threadIdx.x & 31) == 0) s_z[threadIdx.x >> 5] = wz;
    __syncthreads();
    if (threadIdx.x == 0) {
        double bz = 0.0;
        for (int w = 0; w < 8; w++) bz = __dadd_rn(bz, s_z[w]);
        zblock[blockIdx.x] = bz;
        __threadfence();
        s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x < 32) {
        __threadfence();
        const double tot = fixed_sum(zblock, gridDim.x);
        if (threadIdx.x == 0) {
            *z_out = tot;
            *ticket = 0;
        }
    }
}

}  // namespace bh

using namespace bh;

extern "C" int bh_repulsive_f64(const bh_tree_t *t, const bh_bounds_t *bounds,
                                double theta, const double *y_query,
                                int64_t t_begin, int64_t t_end, int sorted_out,
                                double *rep, double *zpart, double *zblock,
                                double *z_out, int32_t *counts, void *ws,
                                size_t ws_bytes, bh_stream_t stream) {
    BH_REQUIRE(theta >= 0, "theta must be >= 0, got %g", theta);
    BH_REQUIRE(t->precision == 64, "bh_repulsive_f64 needs a precision-64 tree");
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
    const RepArgs64 A{(const void *)t->node, (const double2 *)t->ys, t->order,
                      (const double2 *)y_query, bounds, t->status, theta,
                      t_begin, t_end, sorted_out, (double2 *)rep, zpart,
                      (int4 *)counts, zblock, ticket, z_out};
#define BH_REP64(D, CNT, Q)                                                   \
    BH_LAUNCH("k_repulsive64", (k_repulsive64<D, CNT, Q>), grid, kRepThreads, 0, st, A)
#define BH_REP64_2(D)                                                         \
    if (y_query) {                                                            \
        if (counts) BH_REP64(D, true, true); else BH_REP64(D, false, true);   \
    } else {                                                                  \
        if (counts) BH_REP64(D, true, false); else BH_REP64(D, false, false); \
    }
    if (t->code_bits == 32) {
        BH_REP64_2(16)
    } else if (t->code_bits == 64) {
        BH_REP64_2(32)
    } else {
        return set_error(BH_ERR_UNSUPPORTED, "code_bits must be 32 or 64");
    }
#undef BH_REP64
#undef BH_REP64_2
    return BH_OK;
}

extern "C" int bh_attractive_f64(const int64_t *row_ptr, const int32_t *col,
                                 const double *val, int64_t n_rows, int padded,
                                 const double *y, int64_t row_begin,
                                 int64_t row_end, double exaggeration,
                                 const bh_sched_t *sched, double *attr,
                                 bh_stream_t stream) {
    BH_REQUIRE(row_begin >= 0 && row_end <= n_rows && row_begin <= row_end,
               "bad row range");
    if (row_end == row_begin) return BH_OK;
    constexpr int G = 16;
    const int grid = bh_blocks(row_end - row_begin, 256 / G);
    cudaStream_t st = bh_cs(stream);
    const AttArgs64 A{row_ptr, col, val, (const double2 *)y, row_begin,
                      row_end, exaggeration, sched, (double2 *)attr};
    if (padded)
        BH_LAUNCH("k_attractive64", (k_attractive64<G, true>), grid, 256, 0, st, A);
    else
        BH_LAUNCH("k_attractive64", (k_attractive64<G, false>), grid, 256, 0, st, A);
    return BH_OK;
}

extern "C" int bh_forces_f64(const bh_tree_t *t, const bh_bounds_t *bounds,
                             double theta, int64_t t_begin, int64_t t_end,
                             int sorted_out, double *rep, double *zblock,
                             double *z_out, void *ws, size_t ws_bytes,
                             const int64_t *row_ptr, const int32_t *col,
                             const double *val, int64_t n_rows, int padded,
                             const double *y, int64_t row_begin,
                             int64_t row_end, double exaggeration,
                             const bh_sched_t *sched, double *attr,
                             bh_stream_t stream) {
    BH_REQUIRE(theta >= 0, "theta must be >= 0, got %g", theta);
    BH_REQUIRE(t->precision == 64, "bh_forces_f64 needs a precision-64 tree");
    BH_REQUIRE(t_begin >= 0 && t_end <= t->n_points && t_begin <= t_end,
               "bad point range");
    BH_REQUIRE(row_begin >= 0 && row_end <= n_rows && row_begin <= row_end,
               "bad row range");
    if (t_end == t_begin || row_end == row_begin) {
        int rc = bh_attractive_f64(row_ptr, col, val, n_rows, padded, y,
                                   row_begin, row_end, exaggeration, sched,
                                   attr, stream);
        if (rc != BH_OK) return rc;
        return bh_repulsive_f64(t, bounds, theta, nullptr, t_begin, t_end,
                                sorted_out, rep, nullptr, zblock, z_out,
                                nullptr, ws, ws_bytes, stream);
    }
    BH_REQUIRE(ws_bytes >= bh_repulsive_workspace_bytes(t_end - t_begin),
               "repulsive workspace too small");
    constexpr int G = 16;
    const int64_t nr = rep_grid(t_end - t_begin);
    const int64_t na = std::max<int64_t>(
        1, std::min<int64_t>((nr + 1) / 2,
                             bh_blocks(row_end - row_begin, kRepThreads / G)));
    char *w = (char *)ws;
    if (!zblock) zblock = (double *)w;
    unsigned *ticket = (unsigned *)(w + bh_align(sizeof(double) * nr));
    const RepArgs64 R{(const void *)t->node, (const double2 *)t->ys, t->order,
                      nullptr, bounds, t->status, theta, t_begin, t_end,
                      sorted_out, (double2 *)rep, nullptr, nullptr, zblock,
                      ticket, z_out};
    const AttArgs64 A{row_ptr, col, val, (const double2 *)y, row_begin,
                      row_end, exaggeration, sched, (double2 *)attr};
    cudaStream_t st = bh_cs(stream);
    const unsigned grid = (unsigned)(nr + na);
#define BH_FORCES64(D)                                                        \
    if (padded)                                                               \
        BH_LAUNCH("k_forces64", (k_forces64<D, G, true>), grid, kRepThreads,  \
                  0, st, R, A, nr, na);                                       \
    else                                                                      \
        BH_LAUNCH("k_forces64", (k_forces64<D, G, false>), grid, kRepThreads, \
                  0, st, R, A, nr, na);
    if (t->code_bits == 32) {
        BH_FORCES64(16)
    } else if (t->code_bits == 64) {
        BH_FORCES64(32)
    } else {
        return set_error(BH_ERR_UNSUPPORTED, "code_bits must be 32 or 64");
    }
#undef BH_FORCES64
    return BH_OK;
}

extern "C" int bh_repulsive_exact_f64(const double *y, int64_t n, double *rep,
                                      double *zpart, double *z_out, void *ws,
                                      size_t ws_bytes, bh_stream_t stream) {
    BH_REQUIRE(n >= 2, "need at least 2 points");
    BH_REQUIRE(ws_bytes >= bh_repulsive_exact_workspace_bytes(n),
               "exact workspace too small");
    const int grid = bh_blocks(n, 256);
    char *w = (char *)ws;
    k_repulsive_exact64<<<grid, 256, 0, bh_cs(stream)>>>(
        (const double2 *)y, n, (double2 *)rep, zpart, (double *)w,
        (unsigned *)(w + bh_align(sizeof(double) * grid)), z_out);
    BH_CHECK_LAUNCH("k_repulsive_exact64");
    return BH_OK;
}

// ---------------------------------------------------------------------------
// Engine entry points in f64 (bh_step_attractive / bh_step_forces, forces.cu).
// ---------------------------------------------------------------------------
extern "C" int bh_step_attractive_f64(const int64_t *row_ptr,
                                      const int32_t *col, const double *val,
                                      int padded, const double *y,
                                      const bh_part_t *part, int64_t max_rows,
                                      const bh_sched_t *sched, double *attr,
                                      bh_stream_t stream) {
    BH_REQUIRE(part && sched, "part and sched are required");
    if (max_rows <= 0) return BH_OK;
    constexpr int G = 16;
    const AttArgs64 A{row_ptr, col, val, (const double2 *)y, 0, 0, 1.0, sched,
                      (double2 *)attr, part, 0};
    const int grid = bh_blocks(max_rows, 256 / G);
    if (padded)
        BH_LAUNCH("k_attractive64", (k_attractive64<G, true>), grid, 256, 0,
                  bh_cs(stream), A);
    else
        BH_LAUNCH("k_attractive64", (k_attractive64<G, false>), grid, 256, 0,
                  bh_cs(stream), A);
    BH_CHECK_LAUNCH("k_attractive64");
    return BH_OK;
}

extern "C" int bh_step_forces_f64(const bh_tree_t *t,
                                  const bh_bounds_t *bounds, double theta,
                                  const double *y, const int32_t *rank,
                                  const int32_t *qlist, const bh_part_t *part,
                                  int64_t max_points, int mode, double *rep,
                                  double *zpart, void *ws, size_t ws_bytes,
                                  const int64_t *row_ptr, const int32_t *col,
                                  const double *val, int padded,
                                  const bh_sched_t *sched, double *attr,
                                  bh_stream_t stream) {
    BH_REQUIRE(theta >= 0, "theta must be >= 0, got %g", theta);
    BH_REQUIRE(t->precision == 64, "bh_step_forces_f64 needs a precision-64 tree");
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
    const RepArgs64 R{(const void *)t->node, (const double2 *)t->ys, t->order,
                      (const double2 *)y, bounds, t->status, theta, 0,
                      t->n_points, 0, (double2 *)rep, zpart, nullptr,
                      nullptr, ticket, nullptr, part, rank, qlist};
    const AttArgs64 A{row_ptr, col, val, (const double2 *)y, 0, 0, 1.0, sched,
                      (double2 *)attr, part, 1};
    cudaStream_t st = bh_cs(stream);
    if (mode == 2) {
        const int grid = bh_blocks(max_points, 256 / G);
        if (padded)
            BH_LAUNCH("k_attractive64", (k_attractive64<G, true>), grid, 256,
                      0, st, A);
        else
            BH_LAUNCH("k_attractive64", (k_attractive64<G, false>), grid, 256,
                      0, st, A);
        BH_CHECK_LAUNCH("k_attractive64");
        return BH_OK;
    }
    const int64_t na = std::max<int64_t>(
        1, std::min<int64_t>((nr + 1) / 2, bh_blocks(max_points, kRepThreads / G)));
#define BH_STEP64(D)                                                          \
    if (mode == 1)                                                            \
        BH_LAUNCH("k_repulsive64", (k_repulsive64<D, false, false>), (int)nr, \
                  kRepThreads, 0, st, R);                                     \
    else if (padded)                                                          \
        BH_LAUNCH("k_forces64", (k_forces64<D, G, true>), (unsigned)(nr + na),\
                  kRepThreads, 0, st, R, A, nr, na);                          \
    else                                                                      \
        BH_LAUNCH("k_forces64", (k_forces64<D, G, false>),                    \
                  (unsigned)(nr + na), kRepThreads, 0, st, R, A, nr, na);
    if (t->code_bits == 32) {
        BH_STEP64(16)
    } else if (t->code_bits == 64) {
        BH_STEP64(32)
    } else {
        return set_error(BH_ERR_UNSUPPORTED, "code_bits must be 32 or 64");
    }
#undef BH_STEP64
    BH_CHECK_LAUNCH("k_forces64");
    return BH_OK;
}
