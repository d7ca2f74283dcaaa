// Work partition and row exchange plumbing of the multi-GPU engine
// (SURVEY.md 8(e)): every GPU owns a contiguous range of storage slots (the
// Morton order of the last relabel), balanced by cost, and the ranges are
// kept on the device (bh_part_t) so captured CUDA graphs survive a
// re-balance.  The reference has no counterpart (its only parallel axis is
// numba prange over points, optimizer.py:273-286, forces.py:89).
#include "forces.cuh"

namespace bh {

constexpr int kAlign = BH_REP_POINTS_PER_PARTIAL;  // Z partials stay aligned

// Cuts c_0 = 0 < c_1 < ... < c_world = n at multiples of kAlign, c_r the
// smallest aligned slot whose cost prefix reaches r/world of the total; the
// cost of slot s is w_point + its CSR row length, so the prefix is
// w_point * s + row_ptr[s] (row_ptr is the nnz prefix).  Falls back to
// equal shares when a balanced range would exceed `cap` slots.
__global__ void k_partition(const int64_t *__restrict__ rp, int64_t n,
                            int world, double w_point, double split_frac,
                            int64_t cap, int64_t *__restrict__ cuts,
                            bh_part_t *__restrict__ parts) {
    __shared__ int64_t s_cut[65];
    __shared__ int s_ok;
    const int r = threadIdx.x;
    const int64_t nal = (n + kAlign - 1) / kAlign;  // aligned blocks
    const double total = w_point * (double)n + (double)rp[n];
    if (r == 0) s_ok = 1;
    if (r <= world) {
        int64_t c;
        if (r == 0) {
            c = 0;
        } else if (r == world) {
            c = n;
        } else {
            const double want = total * (double)r / (double)world;
            int64_t a = 0, b = nal;  // smallest block index with prefix >= want
            while (a < b) {
                const int64_t m = (a + b) >> 1;
                const int64_t s = m * kAlign < n ? m * kAlign : n;
                const double pre = w_point * (double)s + (double)rp[s];
                if (pre >= want) b = m; else a = m + 1;
            }
            c = a * kAlign < n ? a * kAlign : n;
        }
        s_cut[r] = c;
    }
    __syncthreads();
    if (r < world && s_cut[r + 1] - s_cut[r] > cap) s_ok = 0;
    __syncthreads();
    if (!s_ok && r <= world) {
        const int64_t eq = ((n + world - 1) / world + kAlign - 1) / kAlign * kAlign;
        const int64_t c = (int64_t)r * eq;
        s_cut[r] = r == world ? n : (c < n ? c : n);
    }
    __syncthreads();
    if (r <= world) cuts[r] = s_cut[r];
    if (r < world) {
        const int64_t lo = s_cut[r], hi = s_cut[r + 1];
        bh_part_t p;
        p.lo = lo;
        p.hi = hi;
        p.split = lo + (int64_t)(split_frac * (double)(hi - lo));
        p.world = world;
        parts[r] = p;
    }
}

template <typename E>
__global__ void k_pack(const E *__restrict__ src, const bh_part_t *__restrict__ p,
                       E *__restrict__ dst) {
    const int64_t lo = p->lo, len = p->hi - p->lo;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[lo + i];
}

// dst[cuts[r] + j] = gbuf[r * cap + j] for j < cuts[r+1] - cuts[r]
template <typename E>
__global__ void k_unpack(const E *__restrict__ gbuf, int64_t cap,
                         const int64_t *__restrict__ cuts, int world,
                         E *__restrict__ dst) {
    const int64_t total = cap * world;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / cap);
        const int64_t j = i - (int64_t)r * cap, lo = cuts[r];
        BH_DASSERT(cuts[r + 1] - lo <= cap);
        if (j < cuts[r + 1] - lo) dst[lo + j] = gbuf[i];
    }
}

// Z partial of each 128-slot block of the share, in a fixed order (one warp
// per block: lane l sums slots l, l+32, l+64, l+96 of it, then a butterfly)
// -- the same blocks and sums on any number of GPUs; with z_out (one GPU)
// the last CTA folds all blocks (cta_fold, as bh_sum_partials does after
// the all-reduce on several).
__global__ void __launch_bounds__(kFoldThreads)
k_zsum(const double *__restrict__ zpart, const bh_part_t *__restrict__ p,
       int64_t n, double *__restrict__ zblock, double *__restrict__ z_out,
       unsigned *__restrict__ ticket) {
    __shared__ double s_w[kFoldThreads / 32];
    __shared__ bool s_last;
    const int64_t lo = p->lo, hi = p->hi;
    const int64_t b0 = lo / kAlign, nb = (hi - lo + kAlign - 1) / kAlign;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kW = kFoldThreads / 32;
    for (int64_t q = (int64_t)blockIdx.x * kW + warp; q < nb;
         q += (int64_t)gridDim.x * kW) {
        const int64_t base = (b0 + q) * kAlign;
        double v = 0.0;
#pragma unroll
        for (int r = 0; r < kAlign / 32; r++) {
            const int64_t s = base + r * 32 + lane;
            if (s < hi) v = __dadd_rn(v, zpart[s]);
        }
        v = warp_sum(v);
        if (lane == 0) zblock[b0 + q] = v;
    }
    if (!z_out) return;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const double tot = cta_fold(zblock, (n + kAlign - 1) / kAlign, s_w);
    if (threadIdx.x == 0) {
        *z_out = tot;
        *ticket = 0;
    }
}

// The share's slots in the current sorted order: qlist = the entries of
// order[] that fall in [lo, hi), stable (count / scan / fill over tiles).
constexpr int kQTile = 1024;

__global__ void __launch_bounds__(kQTile)
k_qcount(const int32_t *__restrict__ order, int64_t n,
         const bh_part_t *__restrict__ p, int32_t *__restrict__ counts) {
    __shared__ int s_c[kQTile / 32];
    const int64_t t = blockIdx.x * (int64_t)kQTile + threadIdx.x;
    const int64_t lo = p->lo, hi = p->hi;
    bool in = false;
    if (t < n) {
        const int32_t s = order[t];
        in = s >= lo && s < hi;
    }
    const unsigned m = __ballot_sync(0xffffffffu, in);
    if ((threadIdx.x & 31) == 0) s_c[threadIdx.x >> 5] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        int c = 0;
        for (int i = 0; i < kQTile / 32; i++) c += s_c[i];
        counts[blockIdx.x] = c;
    }
}

__global__ void __launch_bounds__(1024)
k_qscan(int32_t *__restrict__ counts, int64_t ntiles) {
    __shared__ int32_t s_tmp[32];
    __shared__ int32_t s_tot;
    int32_t carry = 0;
    for (int64_t base = 0; base < ntiles; base += 1024) {
        const int64_t i = base + threadIdx.x;
        const int32_t v = i < ntiles ? counts[i] : 0;
        const int32_t ex = block_exclusive_scan(v, s_tmp, &s_tot);
        if (i < ntiles) counts[i] = carry + ex;
        carry += s_tot;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kQTile)
k_qfill(const int32_t *__restrict__ order, int64_t n,
        const bh_part_t *__restrict__ p, const int32_t *__restrict__ offs,
        int32_t *__restrict__ qlist) {
    __shared__ int32_t s_tmp[32];
    __shared__ int32_t s_tot;
    const int64_t t = blockIdx.x * (int64_t)kQTile + threadIdx.x;
    const int64_t lo = p->lo, hi = p->hi;
    int32_t s = 0;
    bool in = false;
    if (t < n) {
        s = order[t];
        in = s >= lo && s < hi;
    }
    const int32_t ex = block_exclusive_scan((int32_t)in, s_tmp, &s_tot);
    if (in) qlist[offs[blockIdx.x] + ex] = s;
}

static int rows_grid(int64_t n) {
    const int64_t b = (n + 255) / 256;
    return (int)(b < 1 ? 1 : (b > kSMs * 8 ? kSMs * 8 : b));
}

}  // namespace bh

using namespace bh;

extern "C" int bh_partition(const int64_t *row_ptr, int64_t n, int world,
                            double w_point, double split_frac, int64_t cap,
                            int64_t *cuts, bh_part_t *parts,
                            bh_stream_t stream) {
    BH_REQUIRE(world >= 1 && world <= 64, "world must be in [1, 64]");
    BH_REQUIRE(n >= 1, "need at least one point");
    BH_REQUIRE(split_frac >= 0.0 && split_frac <= 1.0,
               "split_frac must be in [0, 1]");
    int64_t eq = ((n + world - 1) / world + kAlign - 1) / kAlign * kAlign;
    if (eq > n) eq = n;
    BH_REQUIRE(cap >= eq, "cap %lld below the equal share %lld",
               (long long)cap, (long long)eq);
    k_partition<<<1, 96, 0, bh_cs(stream)>>>(row_ptr, n, world, w_point,
                                             split_frac, cap, cuts, parts);
    BH_CHECK_LAUNCH("k_partition");
    return BH_OK;
}

extern "C" int bh_pack_rows(const void *src, const bh_part_t *part,
                            int64_t cap, int elem_bytes, void *dst,
                            bh_stream_t stream) {
    const int grid = rows_grid(cap);
    cudaStream_t st = bh_cs(stream);
    if (elem_bytes == 8)
        k_pack<uint2><<<grid, 256, 0, st>>>((const uint2 *)src, part, (uint2 *)dst);
    else if (elem_bytes == 16)
        k_pack<uint4><<<grid, 256, 0, st>>>((const uint4 *)src, part, (uint4 *)dst);
    else if (elem_bytes == 4)
        k_pack<uint32_t><<<grid, 256, 0, st>>>((const uint32_t *)src, part, (uint32_t *)dst);
    else
        return set_error(BH_ERR_ARG, "elem_bytes must be 4, 8 or 16");
    BH_CHECK_LAUNCH("k_pack");
    return BH_OK;
}

extern "C" int bh_unpack_rows(const void *gbuf, int64_t cap,
                              const int64_t *cuts, int world, int elem_bytes,
                              void *dst, bh_stream_t stream) {
    const int grid = rows_grid(cap * world);
    cudaStream_t st = bh_cs(stream);
    if (elem_bytes == 8)
        k_unpack<uint2><<<grid, 256, 0, st>>>((const uint2 *)gbuf, cap, cuts, world, (uint2 *)dst);
    else if (elem_bytes == 16)
        k_unpack<uint4><<<grid, 256, 0, st>>>((const uint4 *)gbuf, cap, cuts, world, (uint4 *)dst);
    else if (elem_bytes == 4)
        k_unpack<uint32_t><<<grid, 256, 0, st>>>((const uint32_t *)gbuf, cap, cuts, world, (uint32_t *)dst);
    else
        return set_error(BH_ERR_ARG, "elem_bytes must be 4, 8 or 16");
    BH_CHECK_LAUNCH("k_unpack");
    return BH_OK;
}

extern "C" size_t bh_step_zsum_workspace_bytes(int64_t n) { return 256; }

extern "C" int bh_step_zsum(const double *zpart, const bh_part_t *part,
                            int64_t n, int64_t max_points, double *zblock,
                            double *z_out, void *ws, size_t ws_bytes,
                            bh_stream_t stream) {
    BH_REQUIRE(ws_bytes >= 256, "zsum workspace too small");
    BH_REQUIRE(max_points >= 1 && max_points <= n, "bad max_points");
    const int64_t blocks = (max_points + kAlign - 1) / kAlign;
    int grid = (int)((blocks + kFoldThreads / 32 - 1) / (kFoldThreads / 32));
    if (grid > kSMs * 4) grid = kSMs * 4;
    k_zsum<<<grid, kFoldThreads, 0, bh_cs(stream)>>>(zpart, part, n, zblock,
                                                     z_out, (unsigned *)ws);
    BH_CHECK_LAUNCH("k_zsum");
    return BH_OK;
}

extern "C" size_t bh_step_qlist_workspace_bytes(int64_t n) {
    return bh_align(sizeof(int32_t) * ((n + kQTile - 1) / kQTile)) + 256;
}

extern "C" int bh_step_qlist(const int32_t *order, int64_t n,
                             const bh_part_t *part, int32_t *qlist, void *ws,
                             size_t ws_bytes, bh_stream_t stream) {
    BH_REQUIRE(ws_bytes >= bh_step_qlist_workspace_bytes(n),
               "qlist workspace too small");
    const int64_t ntiles = (n + kQTile - 1) / kQTile;
    int32_t *counts = (int32_t *)ws;
    cudaStream_t st = bh_cs(stream);
    k_qcount<<<(unsigned)ntiles, kQTile, 0, st>>>(order, n, part, counts);
    k_qscan<<<1, 1024, 0, st>>>(counts, ntiles);
    k_qfill<<<(unsigned)ntiles, kQTile, 0, st>>>(order, n, part, counts, qlist);
    BH_CHECK_LAUNCH("k_qfill");
    return BH_OK;
}
