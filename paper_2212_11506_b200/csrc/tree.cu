// Quadtree build and summarize over Morton-sorted codes.
//
// Replaces build_tree (quadtree.py:399-478: serial BFS top + per-subtree
// count/fill with binary searches on 2-bit digits) and summarize
// (quadtree.py:481-519: one parallel pass per level, deepest first).
//
// The reference tree is canonical: nodes of a level are
// sorted by first point, children of a node are consecutive in the next
// level.  With same[t] = number of leading 2-bit digits shared by sorted
// codes t-1 and t (-1 at both ends), point t is the first point of exactly
// one node on every level d in [same[t]+1, min(D, 1+max(same[t], same[t+1]))]
// and node (d, t) is a leaf iff same[t+1] < d or d == D.  A node's id is
// level_off[d] + (number of points before t that start a level-d node), so
// the whole topology is one prefix count over the sorted codes:
//   k_tree_count  per-CTA level histograms (warp ballots)
//   k_tree_emit   per CTA: its level offsets from the counts of the lower
//                 CTAs and the level totals (level_off, M, capacity check);
//                 per point: node ids by ballot-popc ranks, parents, and the
//                 complete record of every single-point leaf (its centre of
//                 mass is the point itself: f64 sum of one value / 1)
// Summarize then runs level by level, deepest first (the reference's own
// schedule): a node's children are the consecutive next-level nodes whose
// parent is the node; f64 sums in the reference's child order, so centres
// of mass are bit-identical to the reference's.
#include <algorithm>

#include "common.cuh"

namespace bh {

constexpr int kTreeThreads = 256;
constexpr int kTreeWarps = kTreeThreads / 32;
#ifndef BH_TREE_PPT
#define BH_TREE_PPT 8
#endif
constexpr int kTreePPT = BH_TREE_PPT;  // sub-chunks per CTA
constexpr int kTreeChunk = kTreeThreads * kTreePPT;
constexpr int kSumThreads = 256;
constexpr int kSumBlocks = kSMs * 8;

template <typename K>
__device__ __forceinline__ int same_digits(const K *__restrict__ sc, int64_t t,
                                           int64_t n, int D) {
    if (t <= 0 || t >= n) return -1;
    K x = sc[t] ^ sc[t - 1];
    if (x == 0) return D;
    int lz = sizeof(K) == 4 ? __clz((unsigned)x) : __clzll((unsigned long long)x);
    return lz >> 1;
}

template <typename K, int D>
__global__ void __launch_bounds__(kTreeThreads)
k_tree_count(const K *__restrict__ sc, int64_t n,
             uint32_t *__restrict__ blk_counts) {
    bh_pdl_trigger();  // the successor may launch early (PDL)
    bh_pdl_wait();     // the predecessor's results are visible

    __shared__ uint32_t s_cnt[kTreeWarps][D + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t cnt[D + 1];
#pragma unroll
    for (int d = 0; d <= D; d++) cnt[d] = 0;
    // all chunks' code loads in flight together (unrolled)
    int lo_[kTreePPT], hi_[kTreePPT];
#pragma unroll
    for (int j = 0; j < kTreePPT; j++) {
        int64_t t = (int64_t)blockIdx.x * kTreeChunk + j * kTreeThreads + threadIdx.x;
        lo_[j] = D + 1;
        hi_[j] = -1;
        if (t < n) {
            int s0 = same_digits(sc, t, n, D), s1 = same_digits(sc, t + 1, n, D);
            lo_[j] = s0 + 1;
            hi_[j] = min(D, 1 + max(s0, s1));
        }
    }
#pragma unroll
    for (int j = 0; j < kTreePPT; j++) {
        const int lo = lo_[j], hi = hi_[j];
#pragma unroll
        for (int d = 0; d <= D; d++)
            cnt[d] += __popc(__ballot_sync(0xffffffffu, lo <= d && d <= hi));
    }
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d <= D; d++) s_cnt[warp][d] = cnt[d];
    }
    __syncthreads();
    if (threadIdx.x <= D) {
        uint32_t s = 0;
        for (int w = 0; w < kTreeWarps; w++) s += s_cnt[w][threadIdx.x];
        blk_counts[(size_t)blockIdx.x * (D + 1) + threadIdx.x] = s;
    }
}

template <typename K, int D, typename T>
__global__ void __launch_bounds__(kTreeThreads)
k_tree_emit(const K *__restrict__ sc, const int32_t *__restrict__ order,
            const p2_t<T> *__restrict__ y, int64_t n,
            const uint32_t *__restrict__ blk_counts, int64_t capacity,
            int32_t *__restrict__ level_off, void *__restrict__ node,
            int32_t *__restrict__ parent, int32_t *__restrict__ node_start,
            int32_t *__restrict__ leaf_end, p2_t<T> *__restrict__ ys,
            int32_t *__restrict__ rank, double2 *__restrict__ tile_sum,
            int32_t *__restrict__ status) {
    bh_pdl_trigger();  // the successor may launch early (PDL)
    bh_pdl_wait();     // the predecessor's results are visible

    using Rec = NodeRec<T>;
    __shared__ double2 s_tsum[kTreeWarps];
    double sx = 0.0, sy = 0.0;  // this thread's points, in order (f64)
    __shared__ uint32_t s_bal[kTreeWarps][D + 1];
    __shared__ uint32_t s_woff[kTreeWarps][D + 1];
    __shared__ uint32_t s_carry[D + 1];
    __shared__ int32_t s_base[D + 1];
    __shared__ uint32_t s_pre[D + 1], s_tot[D + 1];
    __shared__ bool s_ok;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // The CTA's node-id offsets (no separate scan launch): per level, the
    // nodes started in the lower blocks (k_tree_count's counts) and in all
    // blocks -- integer sums, any order; level offsets from the totals.
    if (threadIdx.x <= D) {
        s_carry[threadIdx.x] = 0;
        s_pre[threadIdx.x] = 0;
        s_tot[threadIdx.x] = 0;
    }
    __syncthreads();
    for (int d = 0; d <= D; d++) {
        uint32_t pre = 0, tot = 0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += kTreeThreads) {
            const uint32_t c = blk_counts[(size_t)b * (D + 1) + d];
            tot += c;
            pre += b < (int)blockIdx.x ? c : 0u;
        }
        pre = __reduce_add_sync(0xffffffffu, pre);
        tot = __reduce_add_sync(0xffffffffu, tot);
        if (lane == 0 && tot) {
            atomicAdd(&s_tot[d], tot);
            if (pre) atomicAdd(&s_pre[d], pre);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t acc = 0;
        int levels = 0;
        for (int d = 0; d <= D; d++) {
            s_base[d] = (int32_t)(acc < 0x7fffffff ? acc : 0x7fffffff);
            acc += s_tot[d];
            if (s_tot[d]) levels = d + 1;
        }
        const bool ok = acc <= capacity && acc < (int64_t)BH_CHILD_MASK;
        s_ok = ok;
        if (blockIdx.x == 0) {
            for (int d = 0; d <= D; d++) level_off[d] = s_base[d];
            level_off[D + 1] = (int32_t)(acc < 0x7fffffff ? acc : 0x7fffffff);
            level_off[D + 2] = levels;
            *status = ok ? BH_OK : BH_ERR_CAPACITY;
        }
    }
    __syncthreads();
    if (!s_ok) return;
    if (threadIdx.x <= D) s_base[threadIdx.x] += (int32_t)s_pre[threadIdx.x];
    const unsigned lt = lanemask_lt();
    for (int j = 0; j < kTreePPT; j++) {
        int64_t t = (int64_t)blockIdx.x * kTreeChunk + j * kTreeThreads + threadIdx.x;
        int s0 = -1, s1 = -1, lo = D + 1, hi = -1;
        if (t < n) {
            s0 = same_digits(sc, t, n, D);
            s1 = same_digits(sc, t + 1, n, D);
            lo = s0 + 1;
            hi = min(D, 1 + max(s0, s1));
        }
#pragma unroll
        for (int d = 0; d <= D; d++) {
            unsigned b = __ballot_sync(0xffffffffu, lo <= d && d <= hi);
            if (lane == 0) s_bal[warp][d] = b;
        }
        __syncthreads();
        if (threadIdx.x <= D) {
            // per warp: the level's id base of the warp's first lane
            uint32_t s = s_carry[threadIdx.x];
            for (int w = 0; w < kTreeWarps; w++) {
                s_woff[w][threadIdx.x] = (uint32_t)s_base[threadIdx.x] + s;
                s += __popc(s_bal[w][threadIdx.x]);
            }
            s_carry[threadIdx.x] = s;
        }
        __syncthreads();
        if (t < n) {
            // exclusive rank (global node-id base) of t on level d: the id
            // of t's level-d node if t starts one, else that id + 1
            auto base = [&](int d) -> int32_t {
                return (int32_t)s_woff[warp][d] + __popc(s_bal[warp][d] & lt);
            };
            const int32_t pid = order[t];
            const p2_t<T> p = y[pid];
            ys[t] = p;
            sx = __dadd_rn(sx, (double)p.x);
            sy = __dadd_rn(sy, (double)p.y);
            if (rank) rank[pid] = (int32_t)t;
            // one pass over the levels t starts a node on or ends one on
            // (each level's base evaluated once): t starts a node on
            // d in [lo, hi] and is the last point of its node on d in
            // [s1 + 1, hi] -- the node's end (leaf_end holds the end of
            // every node, leaves and internal)
            const int dend = max(s1 + 1, 0);
            int d = min(lo, dend);
            int32_t b = d <= hi ? base(d) : 0;
            int32_t bprev = (d <= hi && d == lo && d > 0) ? base(d - 1) : 0;
            for (; d <= hi; d++) {
                const int32_t bnext = d < hi ? base(d + 1) : 0;
                if (d >= lo) {
                    const int32_t id = b;
                    const bool leaf = (s1 < d) || d == D;
                    parent[id] = d == 0 ? -1 : (d == lo ? bprev - 1 : bprev);
                    node_start[id] = (int32_t)t;
                    if (!leaf) {
                        Rec::store_info(node, id, (uint32_t)bnext);
                    } else if (s1 < D) {
                        // single-point leaf: complete record (quadtree.py:490-498)
                        Rec::store(node, id, p, 1u, BH_LEAF_BIT | (uint32_t)t);
                    } else {
                        // first point of a run of equal codes (depth-D bucket)
                        Rec::store_info(node, id, BH_LEAF_BIT | (uint32_t)t);
                    }
                }
                if (d >= dend) leaf_end[d >= lo ? b : b - 1] = (int32_t)(t + 1);
                bprev = b;
                b = bnext;
            }
        }
        __syncthreads();
    }
    // the tile's f64 sum of its sorted points (prefix summarize): thread
    // sums in point order, then a fixed butterfly and warp order
    if (tile_sum) {
        sx = warp_sum(sx);
        sy = warp_sum(sy);
        if (lane == 0) s_tsum[warp] = make_double2(sx, sy);
        __syncthreads();
        if (threadIdx.x == 0) {
            double a = 0.0, b = 0.0;
            for (int w = 0; w < kTreeWarps; w++) {
                a = __dadd_rn(a, s_tsum[w].x);
                b = __dadd_rn(b, s_tsum[w].y);
            }
            tile_sum[blockIdx.x] = make_double2(a, b);
        }
    }
}

// ---------------------------------------------------------------------------
// Prefix summarize (the engine's f32 path): every node covers a contiguous
// run [start, end) of sorted points, so its count is end - start and its
// centre of mass (S[end] - S[start]) / count with S the f64 prefix sum of
// the sorted points -- all levels in one pass instead of one launch per
// level.  Single-point leaves keep the point itself (from emit) and depth-D
// buckets their in-order f64 mean, as in the reference; an internal node's
// centre differs from the reference's child-by-child f64 sums only by f64
// rounding (|S| eps ~ 1e-8 at C3 scale, far below the f32 spacing of the
// stored value except at coordinates within ~1e-2 of zero).
// ---------------------------------------------------------------------------
constexpr int kPsThreads = kTreeThreads;
constexpr int kPsPPT = kTreeChunk / kPsThreads;  // consecutive points/thread

// S[t] = sum of sorted points before t (f64), per emit tile: the tile's
// prefix (tile sums of emit, fixed-order warp sum) plus a block scan.
template <typename T>
__global__ void __launch_bounds__(kPsThreads)
k_prefix_scan(const p2_t<T> *__restrict__ ys, int64_t n,
              const double2 *__restrict__ tile_sum, double2 *__restrict__ S,
              const int32_t *__restrict__ status) {
    bh_pdl_trigger();  // the successor may launch early (PDL)
    bh_pdl_wait();     // the predecessor's results are visible

    if (*status != BH_OK) return;
    __shared__ double2 s_w[kTreeWarps];
    __shared__ double2 s_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t b = blockIdx.x;
    if (warp == 0) {
        double a = 0.0, c = 0.0;
        for (int64_t i = lane; i < b; i += 32) {
            const double2 v = tile_sum[i];
            a = __dadd_rn(a, v.x);
            c = __dadd_rn(c, v.y);
        }
        a = warp_sum(a);
        c = warp_sum(c);
        if (lane == 0) s_base = make_double2(a, c);
    }
    const int64_t t0 = b * kTreeChunk + (int64_t)threadIdx.x * kPsPPT;
    double2 loc[kPsPPT];
    double ax = 0.0, ay = 0.0;
#pragma unroll
    for (int k = 0; k < kPsPPT; k++) {
        loc[k] = make_double2(ax, ay);  // exclusive, within the thread
        if (t0 + k < n) {
            const p2_t<T> p = ys[t0 + k];
            ax = __dadd_rn(ax, (double)p.x);
            ay = __dadd_rn(ay, (double)p.y);
        }
    }
    // exclusive scan of the thread totals across the block
    double ex = ax, ey = ay;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double ux = __shfl_up_sync(0xffffffffu, ex, o);
        const double uy = __shfl_up_sync(0xffffffffu, ey, o);
        if (lane >= o) {
            ex = __dadd_rn(ex, ux);
            ey = __dadd_rn(ey, uy);
        }
    }
    if (lane == 31) s_w[warp] = make_double2(ex, ey);
    ex = __dsub_rn(ex, ax);  // exclusive within the warp
    ey = __dsub_rn(ey, ay);
    __syncthreads();
    double bx = s_base.x, by = s_base.y;
    for (int w = 0; w < warp; w++) {
        bx = __dadd_rn(bx, s_w[w].x);
        by = __dadd_rn(by, s_w[w].y);
    }
    bx = __dadd_rn(bx, ex);
    by = __dadd_rn(by, ey);
#pragma unroll
    for (int k = 0; k < kPsPPT; k++)
        if (t0 + k <= n)
            S[t0 + k] = make_double2(__dadd_rn(bx, loc[k].x),
                                     __dadd_rn(by, loc[k].y));
    if (t0 + kPsPPT == n)  // n on a thread boundary: S[n] = all points
        S[n] = make_double2(__dadd_rn(bx, ax), __dadd_rn(by, ay));
}

template <typename T>
__global__ void __launch_bounds__(kSumThreads)
k_summarize_prefix(void *__restrict__ node, const int32_t *__restrict__ parent,
                   const int32_t *__restrict__ node_start,
                   const int32_t *__restrict__ node_end,
                   const p2_t<T> *__restrict__ ys,
                   const double2 *__restrict__ S,
                   const int32_t *__restrict__ level_off, int D,
                   const int32_t *__restrict__ status) {
    bh_pdl_trigger();  // the successor may launch early (PDL)
    bh_pdl_wait();     // the predecessor's results are visible

    using Rec = NodeRec<T>;
    if (*status != BH_OK) return;
    const int32_t m_tot = level_off[D + 1];
    for (int32_t nd = blockIdx.x * kSumThreads + threadIdx.x; nd < m_tot;
         nd += gridDim.x * kSumThreads) {
        const uint32_t info = Rec::info(node, nd);
        const int32_t end = node_end[nd];
        if (info & BH_LEAF_BIT) {
            const uint32_t t = info & ~BH_LEAF_BIT;
            const uint32_t cnt = (uint32_t)end - t;
            if (cnt == 1) continue;  // single-point leaf, completed by emit
            double a = 0.0, b = 0.0;  // depth-D bucket: in-order f64 mean
            for (int64_t q = t; q < end; q++) {
                const p2_t<T> p = ys[q];
                a = __dadd_rn(a, (double)p.x);
                b = __dadd_rn(b, (double)p.y);
            }
            Rec::store(node, nd,
                       mk2<T>((T)__ddiv_rn(a, (double)cnt),
                              (T)__ddiv_rn(b, (double)cnt)),
                       cnt, info);
            continue;
        }
        const int32_t start = node_start[nd];
        const uint32_t cnt = (uint32_t)(end - start);
        const uint32_t fc = info & BH_CHILD_MASK;
        uint32_t k = 1;  // children: the consecutive next-level nodes
#pragma unroll
        for (uint32_t c = 1; c < 4; c++)
            if ((int32_t)(fc + c) < m_tot && parent[fc + c] == nd) k = c + 1;
        const double2 se = S[end], ss = S[start];
        Rec::store(node, nd,
                   mk2<T>((T)__ddiv_rn(__dsub_rn(se.x, ss.x), (double)cnt),
                          (T)__ddiv_rn(__dsub_rn(se.y, ss.y), (double)cnt)),
                   cnt, fc | ((k - 1) << BH_NKIDS_SHIFT));
    }
}

// Summarize one level (quadtree.py:481-508).  Internal node: children are
// the consecutive level-(d+1) nodes with parent == node (at most 4);
// mass = sum, com = sum(m_ch * f64(com_ch)) / m in child order.  Leaves
// still open here are depth-D buckets: f64 mean of their points in order.
template <typename T>
__device__ __forceinline__ void summarize_node(
    void *__restrict__ node, const int32_t *__restrict__ parent,
    const int32_t *__restrict__ leaf_end, const p2_t<T> *__restrict__ ys,
    int32_t nd, int d, int D, int32_t hi_next) {
    using Rec = NodeRec<T>;
    do {
        const uint32_t info = Rec::info(node, nd);
        if (info & BH_LEAF_BIT) {
            if (d < D) continue;  // single-point leaf, completed by emit
            const uint32_t t = info & ~BH_LEAF_BIT;
            const int32_t end = leaf_end[nd];
            const uint32_t cnt = (uint32_t)end - t;
            if (cnt == 1) continue;  // completed by emit
            double a = 0.0, b = 0.0;
            for (int64_t q = t; q < end; q++) {
                const p2_t<T> p = ys[q];
                a = __dadd_rn(a, (double)p.x);
                b = __dadd_rn(b, (double)p.y);
            }
            Rec::store(node, nd,
                       mk2<T>((T)__ddiv_rn(a, (double)cnt),
                              (T)__ddiv_rn(b, (double)cnt)),
                       cnt, info);
            continue;
        }
        const uint32_t fc = info & BH_CHILD_MASK;
        uint32_t m = 0, k = 0;
        double a = 0.0, b = 0.0;
#pragma unroll
        for (uint32_t c = 0; c < 4; c++) {
            if ((int32_t)(fc + c) < hi_next && parent[fc + c] == nd) {
                const p2_t<T> cc = Rec::com(node, fc + c);
                const uint32_t mc = Rec::mass(node, fc + c);
                m += mc;
                a = __dadd_rn(a, __dmul_rn((double)mc, (double)cc.x));
                b = __dadd_rn(b, __dmul_rn((double)mc, (double)cc.y));
                k = c + 1;
            }
        }
        Rec::store(node, nd,
                   mk2<T>((T)__ddiv_rn(a, (double)m), (T)__ddiv_rn(b, (double)m)),
                   m, fc | ((k - 1) << BH_NKIDS_SHIFT));
    } while (false);
}

template <typename T>
__global__ void __launch_bounds__(kSumThreads)
k_summarize_level(void *__restrict__ node, const int32_t *__restrict__ parent,
                  const int32_t *__restrict__ leaf_end,
                  const p2_t<T> *__restrict__ ys,
                  const int32_t *__restrict__ level_off, int d, int D,
                  const int32_t *__restrict__ status) {
    bh_pdl_trigger();  // the successor may launch early (PDL)
    bh_pdl_wait();     // the predecessor's results are visible

    if (*status != BH_OK) return;
    const int32_t lo = level_off[d], hi = level_off[d + 1];
    const int32_t hi_next = d < D ? level_off[d + 2] : hi;
    for (int32_t nd = lo + blockIdx.x * kSumThreads + threadIdx.x; nd < hi;
         nd += gridDim.x * kSumThreads)
        summarize_node<T>(node, parent, leaf_end, ys, nd, d, D, hi_next);
}

// Levels dtop..0 (at most 4^dtop nodes each) in ONE CTA, deepest first with
// a CTA barrier between levels: the small top of the tree costs one launch
// instead of dtop + 1.
constexpr int kSumTopThreads = 1024;

template <typename T>
__global__ void __launch_bounds__(kSumTopThreads)
k_summarize_top(void *__restrict__ node, const int32_t *__restrict__ parent,
                const int32_t *__restrict__ leaf_end,
                const p2_t<T> *__restrict__ ys,
                const int32_t *__restrict__ level_off, int dtop, int D,
                const int32_t *__restrict__ status) {
    bh_pdl_trigger();  // the successor may launch early (PDL)
    bh_pdl_wait();     // the predecessor's results are visible

    if (*status != BH_OK) return;
    for (int d = dtop; d >= 0; d--) {
        const int32_t lo = level_off[d], hi = level_off[d + 1];
        const int32_t hi_next = d < D ? level_off[d + 2] : hi;
        for (int32_t nd = lo + threadIdx.x; nd < hi; nd += kSumTopThreads)
            summarize_node<T>(node, parent, leaf_end, ys, nd, d, D, hi_next);
        __syncthreads();
    }
}

struct TreeLayout {
    size_t counts, offs, bar, tsum, S, total;
    int nblk;
};

static TreeLayout tree_layout(int64_t n, int D) {
    TreeLayout L;
    L.nblk = bh_blocks(n, kTreeChunk);
    L.counts = 0;
    L.offs = bh_align(sizeof(uint32_t) * L.nblk * (D + 1));
    L.bar = L.offs + bh_align(sizeof(uint32_t) * L.nblk * (D + 1));
    L.tsum = L.bar + 256;  // emit's tile sums (prefix summarize)
    L.S = L.tsum + bh_align(sizeof(double2) * L.nblk);
    L.total = L.S + bh_align(sizeof(double2) * (n + 1));
    return L;
}

template <typename K, int D, typename T>
static int build_impl(const bh_tree_t *t, const void *y, void *ws,
                      cudaStream_t st) {
    TreeLayout L = tree_layout(t->n_points, D);
    char *w = (char *)ws;
    uint32_t *cnt = (uint32_t *)(w + L.counts);
    const K *sc = (const K *)t->sorted_codes;
    BH_LAUNCH("k_tree_count", (k_tree_count<K, D>), L.nblk, kTreeThreads, 0,
              st, sc, t->n_points, cnt);
    BH_LAUNCH("k_tree_emit", (k_tree_emit<K, D, T>), L.nblk, kTreeThreads, 0, st,
        sc, t->order, (const p2_t<T> *)y, t->n_points, cnt, t->node_capacity,
        t->level_off,
        (void *)t->node, t->parent, t->node_start, t->leaf_end,
        (p2_t<T> *)t->ys, t->rank, (double2 *)(w + L.tsum), t->status);
    return BH_OK;
}

}  // namespace bh

using namespace bh;

extern "C" size_t bh_tree_workspace_bytes(int64_t n, int code_bits) {
    return tree_layout(n, code_bits / 2).total;
}

static bool tree_f64(const bh_tree_t *t) { return t->precision == 64; }

extern "C" int bh_build_tree(const bh_tree_t *t, const void *y, void *ws,
                             size_t ws_bytes, bh_stream_t stream) {
    BH_REQUIRE(t && t->n_points >= 1, "need at least one point");
    BH_REQUIRE(t->n_points < (int64_t)0x7fffffff, "too many points");
    BH_REQUIRE(ws_bytes >= bh_tree_workspace_bytes(t->n_points, t->code_bits),
               "tree workspace too small");
    BH_REQUIRE(t->precision == 0 || t->precision == 32 || t->precision == 64,
               "precision must be 32 or 64, got %d", t->precision);
    cudaStream_t st = bh_cs(stream);
    if (t->code_bits == 32)
        return tree_f64(t) ? build_impl<uint32_t, 16, double>(t, y, ws, st)
                           : build_impl<uint32_t, 16, float>(t, y, ws, st);
    if (t->code_bits == 64)
        return tree_f64(t) ? build_impl<uint64_t, 32, double>(t, y, ws, st)
                           : build_impl<uint64_t, 32, float>(t, y, ws, st);
    return set_error(BH_ERR_UNSUPPORTED, "code_bits must be 32 or 64");
}

extern "C" int bh_summarize(const bh_tree_t *t, void *ws, size_t ws_bytes,
                            bh_stream_t stream) {
    BH_REQUIRE(t && t->n_points >= 1, "need at least one point");
    BH_REQUIRE(ws_bytes >= bh_tree_workspace_bytes(t->n_points, t->code_bits),
               "tree workspace too small");
    const int D = t->max_depth;
    // One launch per level, deepest first: within a CUDA graph these are
    // pipelined back to back (~5 us each at C3), cheaper than a cooperative
    // kernel with grid barriers between levels (measured 133 us vs 80 us).
    static const int max_blocks = [] {  // tuning knob BH_SUM_BLOCKS
        const char *s = getenv("BH_SUM_BLOCKS");
        const int b = s ? atoi(s) : kSumBlocks;
        return b > 0 ? b : kSumBlocks;
    }();
    int grid = bh_blocks(t->n_points, kSumThreads);
    if (grid > max_blocks) grid = max_blocks;
    static const int top = [] {  // tuning knob BH_SUM_TOP (-1: off)
        const char *s = getenv("BH_SUM_TOP");
        return s ? atoi(s) : 6;
    }();
    const int dtop = std::min(top, D);
    for (int d = D; d > dtop; d--) {
        if (tree_f64(t))
            BH_LAUNCH("k_summarize_level", k_summarize_level<double>, grid,
                      kSumThreads, 0, bh_cs(stream), (void *)t->node, t->parent,
                      t->leaf_end, (const double2 *)t->ys, t->level_off, d, D,
                      t->status);
        else
            BH_LAUNCH("k_summarize_level", k_summarize_level<float>, grid,
                      kSumThreads, 0, bh_cs(stream), (void *)t->node, t->parent,
                      t->leaf_end, (const float2 *)t->ys, t->level_off, d, D,
                      t->status);
    }
    if (dtop >= 0) {
        if (tree_f64(t))
            BH_LAUNCH("k_summarize_top", k_summarize_top<double>, 1,
                      kSumTopThreads, 0, bh_cs(stream), (void *)t->node,
                      t->parent, t->leaf_end, (const double2 *)t->ys,
                      t->level_off, dtop, D, t->status);
        else
            BH_LAUNCH("k_summarize_top", k_summarize_top<float>, 1,
                      kSumTopThreads, 0, bh_cs(stream), (void *)t->node,
                      t->parent, t->leaf_end, (const float2 *)t->ys,
                      t->level_off, dtop, D, t->status);
    }
    return BH_OK;
}

extern "C" int bh_summarize_prefix(const bh_tree_t *t, void *ws,
                                   size_t ws_bytes, bh_stream_t stream) {
    BH_REQUIRE(t && t->n_points >= 1, "need at least one point");
    BH_REQUIRE(t->precision != 64,
               "precision-64 tree: use bh_summarize (bit-exact f64 centres)");
    BH_REQUIRE(ws_bytes >= bh_tree_workspace_bytes(t->n_points, t->code_bits),
               "tree workspace too small");
    const TreeLayout L = tree_layout(t->n_points, t->max_depth);
    char *w = (char *)ws;
    const double2 *tsum = (const double2 *)(w + L.tsum);
    double2 *S = (double2 *)(w + L.S);
    cudaStream_t st = bh_cs(stream);
    BH_LAUNCH("k_prefix_scan", k_prefix_scan<float>, L.nblk, kPsThreads, 0,
              st, (const float2 *)t->ys, t->n_points, tsum, S, t->status);
    // about one node per thread (a tree has at most ~n nodes in practice;
    // the grid-stride loop covers any more): the gathers of a node are
    // dependent, so memory-level parallelism comes from threads
    static const int per_thread = [] {  // tuning knob BH_SUMP_NODES
        const char *s = getenv("BH_SUMP_NODES");
        const int v = s ? atoi(s) : 1;
        return v > 0 ? v : 1;
    }();
    const int grid = (int)std::max<int64_t>(
        1, bh_blocks(t->n_points, (int64_t)kSumThreads * per_thread));
    BH_LAUNCH("k_summarize_prefix", k_summarize_prefix<float>, grid,
              kSumThreads, 0, st, (void *)t->node, t->parent, t->node_start,
              t->leaf_end, (const float2 *)t->ys, (const double2 *)S,
              t->level_off, t->max_depth, t->status);
    return BH_OK;
}
