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
//   k_tree_scan   one CTA: per-level scans -> CTA offsets, level_off, M
//   k_tree_emit   per point: node ids by ballot-popc ranks, records, parents
// and summarize is a single bottom-up pass in which the last child to finish
// computes its parent (f64 sums in the reference's child order, so centres of
// mass are bit-identical to the reference's).
#include "common.cuh"

namespace bh {

constexpr int kTreeThreads = 256;
constexpr int kTreeWarps = kTreeThreads / 32;
constexpr int kTreePPT = 8;  // sub-chunks per CTA
constexpr int kTreeChunk = kTreeThreads * kTreePPT;

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
    __shared__ uint32_t s_cnt[kTreeWarps][D + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t cnt[D + 1];
#pragma unroll
    for (int d = 0; d <= D; d++) cnt[d] = 0;
    for (int j = 0; j < kTreePPT; j++) {
        int64_t t = (int64_t)blockIdx.x * kTreeChunk + j * kTreeThreads + threadIdx.x;
        int lo = D + 1, hi = -1;
        if (t < n) {
            int s0 = same_digits(sc, t, n, D), s1 = same_digits(sc, t + 1, n, D);
            lo = s0 + 1;
            hi = min(D, 1 + max(s0, s1));
        }
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

// One CTA of 1024 threads: warp w scans level w's CTA counts.
template <int D>
__global__ void __launch_bounds__(1024)
k_tree_scan(const uint32_t *__restrict__ blk_counts, int nblk,
            uint32_t *__restrict__ blk_off, int32_t *__restrict__ level_off,
            int64_t capacity, int32_t *__restrict__ status) {
    __shared__ uint32_t s_tot[D + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int d = warp; d <= D; d += 32) {
        uint32_t carry = 0;
        for (int b0 = 0; b0 < nblk; b0 += 32) {
            int b = b0 + lane;
            uint32_t v = b < nblk ? blk_counts[(size_t)b * (D + 1) + d] : 0u;
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (b < nblk) blk_off[(size_t)b * (D + 1) + d] = carry + x - v;
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) s_tot[d] = carry;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t acc = 0;
        int levels = 0;
        level_off[0] = 0;
        for (int d = 0; d <= D; d++) {
            acc += s_tot[d];
            if (s_tot[d]) levels = d + 1;
            level_off[d + 1] = (int32_t)(acc < 0x7fffffff ? acc : 0x7fffffff);
        }
        level_off[D + 2] = levels;
        *status = (acc > capacity || acc >= (int64_t)BH_CHILD_MASK) ? BH_ERR_CAPACITY
                                                                    : BH_OK;
    }
}

template <typename K, int D>
__global__ void __launch_bounds__(kTreeThreads)
k_tree_emit(const K *__restrict__ sc, const int32_t *__restrict__ order,
            const float2 *__restrict__ y, int64_t n,
            const uint32_t *__restrict__ blk_off,
            const int32_t *__restrict__ level_off, float4 *__restrict__ node,
            int32_t *__restrict__ parent, int32_t *__restrict__ node_start,
            int32_t *__restrict__ leaf_end, uint32_t *__restrict__ nkids,
            float2 *__restrict__ ys, int32_t *__restrict__ pt_leaf,
            int32_t *__restrict__ rank, const int32_t *__restrict__ status) {
    if (*status != BH_OK) return;
    __shared__ uint32_t s_bal[kTreeWarps][D + 1];
    __shared__ uint32_t s_woff[kTreeWarps][D + 1];
    __shared__ uint32_t s_carry[D + 1];
    __shared__ int32_t s_base[D + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x <= D) {
        s_carry[threadIdx.x] = 0;
        s_base[threadIdx.x] = level_off[threadIdx.x] +
                              (int32_t)blk_off[(size_t)blockIdx.x * (D + 1) + threadIdx.x];
    }
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
            uint32_t s = s_carry[threadIdx.x];
            for (int w = 0; w < kTreeWarps; w++) {
                s_woff[w][threadIdx.x] = s;
                s += __popc(s_bal[w][threadIdx.x]);
            }
            s_carry[threadIdx.x] = s;
        }
        __syncthreads();
        if (t < n) {
            // exclusive rank (global node-id base) of t on level d
            auto base = [&](int d) -> int32_t {
                return s_base[d] + (int32_t)s_woff[warp][d] +
                       __popc(s_bal[warp][d] & lt);
            };
            const int32_t pid = order[t];
            ys[t] = y[pid];
            if (rank) rank[pid] = (int32_t)t;
            int32_t leaf_id = -1;
            for (int d = lo; d <= hi; d++) {
                int32_t id = base(d);
                bool leaf = (s1 < d) || d == D;
                uint32_t info = leaf ? (BH_LEAF_BIT | (uint32_t)t) : (uint32_t)base(d + 1);
                int32_t par = d == 0 ? -1 : (d == lo ? base(d - 1) - 1 : base(d - 1));
                node[id].w = __uint_as_float(info);
                parent[id] = par;
                node_start[id] = (int32_t)t;
                if (par >= 0) atomicAdd(&nkids[par], 1u);
                if (leaf) {
                    leaf_id = id;
                    if (s1 < D) leaf_end[id] = (int32_t)(t + 1);
                }
            }
            pt_leaf[t] = leaf_id;
            // last point of a run of equal codes closes its depth-D leaf
            if (s0 == D && s1 < D) leaf_end[base(D) - 1] = (int32_t)(t + 1);
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256)
k_summarize(float4 *__restrict__ node, const int32_t *__restrict__ parent,
            const int32_t *__restrict__ leaf_end, uint32_t *__restrict__ nkids,
            uint32_t *__restrict__ arrive, const float2 *__restrict__ ys,
            const int32_t *__restrict__ pt_leaf, int64_t n,
            const int32_t *__restrict__ status) {
    if (*status != BH_OK) return;
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    int32_t cur = pt_leaf[t];
    if (cur < 0) return;
    // leaf: f64 mean of its points in sorted order (quadtree.py:490-498)
    int32_t end = leaf_end[cur];
    uint32_t cnt = (uint32_t)(end - t);
    float cx, cy;
    if (cnt == 1) {
        float2 p = ys[t];
        cx = p.x;
        cy = p.y;
    } else {
        double a = 0.0, b = 0.0;
        for (int64_t q = t; q < end; q++) {
            float2 p = ys[q];
            a = __dadd_rn(a, (double)p.x);
            b = __dadd_rn(b, (double)p.y);
        }
        cx = __double2float_rn(__ddiv_rn(a, (double)cnt));
        cy = __double2float_rn(__ddiv_rn(b, (double)cnt));
    }
    node[cur] = make_float4(cx, cy, __uint_as_float(cnt),
                            __uint_as_float(BH_LEAF_BIT | (uint32_t)t));
    // internal: mass-weighted f64 mean of the children, child order
    // (quadtree.py:499-508); the last child to arrive computes the parent
    while (true) {
        int32_t p = parent[cur];
        if (p < 0) break;
        __threadfence();
        uint32_t got = atomicAdd(&arrive[p], 1u) + 1;
        // read after the arrival: only the last child can see the full
        // count; an earlier child may see it or the last child's reset (0)
        uint32_t k = __ldcg(&nkids[p]);
        if (got != k) break;
        __threadfence();
        uint32_t fc = __float_as_uint(node[p].w) & BH_CHILD_MASK;
        uint32_t m = 0;
        double a = 0.0, b = 0.0;
        for (uint32_t c = 0; c < k; c++) {
            float4 r = __ldcg(&node[fc + c]);
            uint32_t mc = __float_as_uint(r.z);
            m += mc;
            a = __dadd_rn(a, __dmul_rn((double)mc, (double)r.x));
            b = __dadd_rn(b, __dmul_rn((double)mc, (double)r.y));
        }
        node[p] = make_float4(__double2float_rn(__ddiv_rn(a, (double)m)),
                              __double2float_rn(__ddiv_rn(b, (double)m)),
                              __uint_as_float(m),
                              __uint_as_float(fc | ((k - 1) << BH_NKIDS_SHIFT)));
        arrive[p] = 0;
        nkids[p] = 0;
        cur = p;
    }
}

struct TreeLayout {
    size_t counts, offs, total;
    int nblk;
};

static TreeLayout tree_layout(int64_t n, int D) {
    TreeLayout L;
    L.nblk = bh_blocks(n, kTreeChunk);
    L.counts = 0;
    L.offs = bh_align(sizeof(uint32_t) * L.nblk * (D + 1));
    L.total = L.offs + bh_align(sizeof(uint32_t) * L.nblk * (D + 1));
    return L;
}

template <typename K, int D>
static int build_impl(const bh_tree_t *t, const float *y, void *ws,
                      cudaStream_t st) {
    TreeLayout L = tree_layout(t->n_points, D);
    char *w = (char *)ws;
    uint32_t *cnt = (uint32_t *)(w + L.counts), *off = (uint32_t *)(w + L.offs);
    const K *sc = (const K *)t->sorted_codes;
    k_tree_count<K, D><<<L.nblk, kTreeThreads, 0, st>>>(sc, t->n_points, cnt);
    BH_CHECK_LAUNCH("k_tree_count");
    k_tree_scan<D><<<1, 1024, 0, st>>>(cnt, L.nblk, off, t->level_off,
                                       t->node_capacity, t->status);
    BH_CHECK_LAUNCH("k_tree_scan");
    k_tree_emit<K, D><<<L.nblk, kTreeThreads, 0, st>>>(
        sc, t->order, (const float2 *)y, t->n_points, off, t->level_off,
        (float4 *)t->node, t->parent, t->node_start, t->leaf_end, t->nkids,
        (float2 *)t->ys, t->pt_leaf, t->rank, t->status);
    BH_CHECK_LAUNCH("k_tree_emit");
    return BH_OK;
}

}  // namespace bh

using namespace bh;

extern "C" size_t bh_tree_workspace_bytes(int64_t n, int code_bits) {
    return tree_layout(n, code_bits / 2).total;
}

extern "C" int bh_build_tree(const bh_tree_t *t, const float *y, void *ws,
                             size_t ws_bytes, bh_stream_t stream) {
    BH_REQUIRE(t && t->n_points >= 1, "need at least one point");
    BH_REQUIRE(t->n_points < (int64_t)0x7fffffff, "too many points");
    BH_REQUIRE(ws_bytes >= bh_tree_workspace_bytes(t->n_points, t->code_bits),
               "tree workspace too small");
    if (t->code_bits == 32) return build_impl<uint32_t, 16>(t, y, ws, bh_cs(stream));
    if (t->code_bits == 64) return build_impl<uint64_t, 32>(t, y, ws, bh_cs(stream));
    return set_error(BH_ERR_UNSUPPORTED, "code_bits must be 32 or 64");
}

extern "C" int bh_summarize(const bh_tree_t *t, bh_stream_t stream) {
    BH_REQUIRE(t && t->n_points >= 1, "need at least one point");
    k_summarize<<<bh_blocks(t->n_points, 256), 256, 0, bh_cs(stream)>>>(
        (float4 *)t->node, t->parent, t->leaf_end, t->nkids, t->arrive,
        (const float2 *)t->ys, t->pt_leaf, t->n_points, t->status);
    BH_CHECK_LAUNCH("k_summarize");
    return BH_OK;
}
