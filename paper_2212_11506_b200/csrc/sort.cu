// Stable LSD radix sort of (key, uint32 payload) pairs -- the on-device
// replacement of _radix_argsort (quadtree.py:188-227).
//
// One histogram pass computes every 8-bit digit histogram at once; then one
// "onesweep" kernel per digit: each CTA claims a tile in launch order, ranks
// its keys per digit with warp ballots (stable: tile order = index order),
// publishes its per-digit counts and resolves its global offsets with a
// decoupled look-back over the previous tiles, stages the tile in shared
// memory in output order and writes coalesced runs.  Stability makes the
// permutation equal to np.argsort(keys, kind="stable").
#include "common.cuh"

namespace bh {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr uint32_t kFlagA = 1u << 30, kFlagP = 2u << 30, kValMask = (1u << 30) - 1;
#ifndef BH_SORT_LOOKBACK
// predecessors polled per round trip: 4 measured best at C3 (16: +7%,
// 32: +2x; the pass is bound by per-tile latency over ~2 waves of tiles)
#define BH_SORT_LOOKBACK 4
#endif
constexpr int kLookback = BH_SORT_LOOKBACK;

#ifndef BH_SORT_IPT32
// keys per thread for 32-bit keys: 12 (3072-key tiles, 424 tiles at C3)
// measured best (sort + build 168 us vs 186 us at 8, 184 at 16)
#define BH_SORT_IPT32 12
#endif
template <typename K>
struct SortCfg {
    static constexpr int IPT = sizeof(K) == 4 ? BH_SORT_IPT32 : 12;
    static constexpr int TILE = kSortThreads * IPT;
    static constexpr size_t SMEM = (size_t)TILE * (sizeof(K) + 4);
    static_assert(SMEM <= 48 * 1024, "tile must fit the default smem limit");
};

// Digit histograms of all passes, and the reset of the passes' control words
// (look-back status, tile counters) -- no memset node in the iteration, so
// the whole chain is kernel-to-kernel (PDL).  Counts accumulate into one of
// two buffers chosen by a call epoch; the last CTA publishes them to `hist`,
// and zeroes the other buffer for the next call.
// Where the histogram pass gets its keys (a functor: the key array of
// bh_sort; a fused key computation was measured and rejected).
template <typename K>
struct KeysIn {
    const K *__restrict__ keys;
    __device__ __forceinline__ K operator()(int64_t i) const { return keys[i]; }
};

template <typename K, typename Src = KeysIn<K>>
__global__ void __launch_bounds__(256)
k_sort_hist(const Src src, int64_t n, int passes,
            uint32_t *__restrict__ hist, uint32_t *__restrict__ acc2,
            uint32_t *__restrict__ epoch, unsigned *__restrict__ ticket,
            uint32_t *__restrict__ zero, int64_t zero_words) {
    bh_pdl_trigger();  // the successor may launch early (PDL)
    bh_pdl_wait();     // the predecessor's results are visible
    const uint32_t ep = *(volatile uint32_t *)epoch;
    uint32_t *acc = acc2 + (size_t)(ep & 1u) * 8 * 256;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
         i < zero_words; i += (int64_t)gridDim.x * blockDim.x)
        zero[i] = 0u;

    __shared__ uint32_t sh[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();
    // Each thread counts a run of kRun consecutive keys with run-length
    // aggregation: the keys arrive nearly sorted (the previous iteration's
    // Morton order), so the high digits change rarely within a run and cost
    // one shared atomic per change instead of one per key.
    constexpr int kRun = 16;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * kRun; s < n;
         s += nthreads * kRun) {
        const int cnt = (int)min((int64_t)kRun, n - s);
        K kk[kRun];
#pragma unroll
        for (int j = 0; j < kRun; j++) kk[j] = j < cnt ? src(s + j) : K(0);
        for (int p = 0; p < passes; p++) {
            unsigned cur = (unsigned)(kk[0] >> (8 * p)) & 0xFFu, run = 1;
#pragma unroll
            for (int j = 1; j < kRun; j++) {
                if (j >= cnt) break;
                const unsigned d = (unsigned)(kk[j] >> (8 * p)) & 0xFFu;
                if (d == cur) {
                    run++;
                } else {
                    atomicAdd(&sh[p][cur], run);
                    cur = d;
                    run = 1;
                }
            }
            atomicAdd(&sh[p][cur], run);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) {
        uint32_t c = (&sh[0][0])[i];
        if (c) atomicAdd(&acc[i], c);
    }
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    uint32_t *other = acc2 + (size_t)((ep + 1u) & 1u) * 8 * 256;
    for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) {
        hist[i] = __ldcg(&acc[i]);
        other[i] = 0u;
    }
    if (threadIdx.x == 0) {
        *epoch = ep + 1u;
        *ticket = 0u;
    }
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads)
k_sort_pass(const K *__restrict__ kin, const uint32_t *__restrict__ vin,
            K *__restrict__ kout, uint32_t *__restrict__ vout, int64_t n,
            int shift, const uint32_t *__restrict__ hist,
            uint32_t *__restrict__ status, uint32_t *__restrict__ tile_ctr) {
    bh_pdl_trigger();  // the successor may launch early (PDL)
    bh_pdl_wait();     // the predecessor's results are visible

    constexpr int IPT = SortCfg<K>::IPT, TILE = SortCfg<K>::TILE;
    extern __shared__ __align__(16) unsigned char smem[];
    K *s_keys = (K *)smem;
    uint32_t *s_vals = (uint32_t *)(s_keys + TILE);
    __shared__ uint32_t s_whist[kSortWarps][256];
    __shared__ uint32_t s_tile_excl[256], s_glob[256], s_scan[32];
    __shared__ uint32_t s_tile, s_total;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
#pragma unroll
    for (int w = 0; w < kSortWarps; w++) s_whist[w][tid] = 0;
    uint32_t h = hist[tid];
    uint32_t hx = block_exclusive_scan<uint32_t>(h, s_scan, &s_total);
    s_glob[tid] = hx;
    __syncthreads();

    const int64_t base = (int64_t)s_tile * TILE;
    const int64_t seg = base + (int64_t)warp * 32 * IPT;
    K k[IPT];
    uint32_t v[IPT], r[IPT];
#pragma unroll
    for (int j = 0; j < IPT; j++) {
        int64_t idx = seg + j * 32 + lane;
        bool ok = idx < n;
        k[j] = ok ? kin[idx] : K(0);
        v[j] = ok ? (vin ? vin[idx] : (uint32_t)idx) : 0u;
    }
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < IPT; j++) {
        int64_t idx = seg + j * 32 + lane;
        bool ok = idx < n;
        unsigned d = (unsigned)(k[j] >> shift) & 0xFFu;
        unsigned peers = __ballot_sync(0xffffffffu, ok);
#pragma unroll
        for (int b = 0; b < 8; b++) {
            unsigned bit = (d >> b) & 1u;
            unsigned bb = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? bb : ~bb;
        }
        uint32_t old = 0;
        if (ok) old = s_whist[warp][d];
        __syncwarp();
        if (ok && lane == __ffs(peers) - 1) s_whist[warp][d] = old + __popc(peers);
        __syncwarp();
        r[j] = old + __popc(peers & lt);
    }
    __syncthreads();

    // per digit: exclusive over warps, then over digits (local positions)
    const int d = tid;
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; w++) {
        uint32_t c = s_whist[w][d];
        s_whist[w][d] = cnt;
        cnt += c;
    }
    uint32_t te = block_exclusive_scan<uint32_t>(cnt, s_scan, &s_total);
    s_tile_excl[d] = te;

    // decoupled look-back for this digit's global offset
    const uint32_t tile = s_tile;
    uint32_t prefix = 0;
    if (tile == 0) {
        st_relaxed(&status[d], kFlagP | cnt);
    } else {
        st_relaxed(&status[(size_t)tile * 256 + d], kFlagA | cnt);
        // look back kLookback predecessors per L2 round trip (the P frontier
        // then advances kLookback tiles per trip); stop at the first
        // inclusive prefix (P), re-poll from the first unpublished one
        int64_t p = (int64_t)tile - 1;
        bool done = false;
        while (!done) {
            uint32_t w[kLookback];
#pragma unroll
            for (int k = 0; k < kLookback; k++)
                w[k] = p - k >= 0 ? ld_relaxed(&status[(size_t)(p - k) * 256 + d]) : 0u;
#pragma unroll
            for (int k = 0; k < kLookback; k++) {
                const uint32_t f = w[k] & ~kValMask;
                if (f == 0) break;
                prefix += w[k] & kValMask;
                p--;
                if (f == kFlagP) {
                    done = true;
                    break;
                }
            }
        }
        st_relaxed(&status[(size_t)tile * 256 + d], kFlagP | (prefix + cnt));
    }
    s_glob[d] += prefix;
    __syncthreads();

#pragma unroll
    for (int j = 0; j < IPT; j++) {
        int64_t idx = seg + j * 32 + lane;
        if (idx < n) {
            unsigned dd = (unsigned)(k[j] >> shift) & 0xFFu;
            uint32_t pos = s_tile_excl[dd] + s_whist[warp][dd] + r[j];
            s_keys[pos] = k[j];
            s_vals[pos] = v[j];
        }
    }
    __syncthreads();
    int64_t rem = n - base;
    const int valid = rem < TILE ? (int)rem : TILE;
    for (int i = tid; i < valid; i += kSortThreads) {
        K kk = s_keys[i];
        unsigned dd = (unsigned)(kk >> shift) & 0xFFu;
        int64_t g = (int64_t)s_glob[dd] + (i - (int)s_tile_excl[dd]);
        kout[g] = kk;
        vout[g] = s_vals[i];
    }
}

struct SortLayout {
    size_t keys_a, vals_a, keys_b, vals_b, hist, ctr, status, acc, misc, total;
    int passes;
    int64_t tiles;
};

template <typename K>
static SortLayout sort_layout(int64_t n, int key_bits) {
    SortLayout L;
    L.passes = (key_bits + 7) / 8;
    L.tiles = (n + SortCfg<K>::TILE - 1) / SortCfg<K>::TILE;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += bh_align(bytes);
        return o;
    };
    L.keys_a = take(sizeof(K) * n);
    L.vals_a = take(4 * n);
    L.keys_b = take(sizeof(K) * n);
    L.vals_b = take(4 * n);
    L.hist = take(4 * 256 * L.passes);
    L.ctr = take(4 * L.passes);
    L.status = take(4 * 256 * (size_t)L.tiles * L.passes);
    L.acc = take(4 * 2 * 8 * 256);  // two histogram accumulators
    L.misc = take(16);              // epoch, ticket
    L.total = off;
    return L;
}

template <typename K, typename Src = KeysIn<K>>
static int sort_impl(const K *keys, const uint32_t *vals, int64_t n,
                     int key_bits, K *out_keys, uint32_t *out_vals, void *ws,
                     size_t ws_bytes, cudaStream_t st, Src src) {
    BH_REQUIRE(n >= 0 && n < (int64_t)kValMask, "sort size out of range");
    BH_REQUIRE(key_bits >= 1 && key_bits <= 8 * (int)sizeof(K),
               "key_bits out of range");
    if (n == 0) return BH_OK;
    SortLayout L = sort_layout<K>(n, key_bits);
    BH_REQUIRE(ws_bytes >= L.total, "sort workspace too small (%zu < %zu)",
               ws_bytes, L.total);
    char *w = (char *)ws;
    uint32_t *hist = (uint32_t *)(w + L.hist);
    uint32_t *ctr = (uint32_t *)(w + L.ctr);
    uint32_t *status = (uint32_t *)(w + L.status);
    uint32_t *misc = (uint32_t *)(w + L.misc);
    int hb = bh_blocks(n, 256 * 16);
    if (hb > kSMs * 4) hb = kSMs * 4;
    // tile counters and look-back status are contiguous: [ctr, status)
    const int64_t zero_words = (int64_t)((L.status - L.ctr) / 4 +
                                         (size_t)256 * L.tiles * L.passes);
    BH_LAUNCH("k_sort_hist", (k_sort_hist<K, Src>), hb, 256, 0, st, src, n,
              L.passes, hist, (uint32_t *)(w + L.acc), misc, misc + 1, ctr,
              zero_words);
    K *kb[2] = {(K *)(w + L.keys_a), (K *)(w + L.keys_b)};
    uint32_t *vb[2] = {(uint32_t *)(w + L.vals_a), (uint32_t *)(w + L.vals_b)};
    for (int p = 0; p < L.passes; p++) {
        const K *ki = p == 0 ? keys : kb[(p - 1) & 1];
        const uint32_t *vi = p == 0 ? vals : vb[(p - 1) & 1];
        K *ko = p == L.passes - 1 ? out_keys : kb[p & 1];
        uint32_t *vo = p == L.passes - 1 ? out_vals : vb[p & 1];
        BH_LAUNCH("k_sort_pass", k_sort_pass<K>, (unsigned)L.tiles,
                  kSortThreads, SortCfg<K>::SMEM, st, ki, vi, ko, vo, n, 8 * p,
                  (const uint32_t *)(hist + 256 * p),
                  status + (size_t)256 * L.tiles * p, ctr + p);
    }
    return BH_OK;
}

}  // namespace bh

using namespace bh;

extern "C" size_t bh_sort_workspace_bytes(int64_t n, int key_bits) {
    return key_bits <= 32 ? sort_layout<uint32_t>(n, key_bits).total
                          : sort_layout<uint64_t>(n, key_bits).total;
}

extern "C" int bh_sort_pairs(const void *keys, const uint32_t *vals, int64_t n,
                             int key_bits, void *sorted_keys,
                             uint32_t *sorted_vals, void *ws, size_t ws_bytes,
                             bh_stream_t stream) {
    if (key_bits <= 32)
        return sort_impl((const uint32_t *)keys, vals, n, key_bits,
                         (uint32_t *)sorted_keys, sorted_vals, ws, ws_bytes,
                         bh_cs(stream),
                         KeysIn<uint32_t>{(const uint32_t *)keys});
    return sort_impl((const uint64_t *)keys, vals, n, key_bits,
                     (uint64_t *)sorted_keys, sorted_vals, ws, ws_bytes,
                     bh_cs(stream), KeysIn<uint64_t>{(const uint64_t *)keys});
}

extern "C" int bh_sort(const void *keys, int64_t n, int key_bits,
                       void *sorted_keys, int32_t *order, void *ws,
                       size_t ws_bytes, bh_stream_t stream) {
    return bh_sort_pairs(keys, nullptr, n, key_bits, sorted_keys,
                         (uint32_t *)order, ws, ws_bytes, stream);
}
