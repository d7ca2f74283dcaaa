// Binary-search perplexity (affinity.py:61-118) and the symmetrised CSR
// (affinity.py:121-158), plus the padded CSR layout used by the attractive
// sweep.  One-time work (before the optimisation loop).
#include <float.h>

#include "common.cuh"

namespace bh {

// ---------------------------------------------------------------------------
// BSP: one warp per row, K distances held in registers (KPL per lane), f64
// bisection with the reference's exact schedule: beta starts at 1, doubles
// while no upper bound is known, else bisects; stop when |H - ln u| <= tol;
// normalisation uses the LAST evaluated s (affinity.py:73-95).  Sums are
// lane-strided partials + a butterfly, so all lanes agree bit for bit and
// take identical branches.
// ---------------------------------------------------------------------------
template <int KPL, typename S>
__global__ void __launch_bounds__(256)
k_bsp(const S *__restrict__ sqd, int64_t n, int k, double ln_u,
      double tol, int max_iter, double *__restrict__ betas,
      double *__restrict__ cond) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t row = wid; row < n; row += nw) {
        const S *r = sqd + row * (int64_t)k;
        double *out = cond + row * (int64_t)k;
        const double dmax = (double)r[k - 1];
        if (dmax <= 0.0) {
            for (int j = lane; j < k; j += 32) out[j] = __ddiv_rn(1.0, (double)k);
            if (lane == 0) betas[row] = 1.0;
            continue;
        }
        const double dmin = (double)r[0];
        double delta[KPL];
#pragma unroll
        for (int j = 0; j < KPL; j++) {
            int idx = lane + 32 * j;
            delta[j] = idx < k ? __dsub_rn((double)r[idx], dmin) : 0.0;
        }
        double beta = 1.0, lo = 0.0, hi = INFINITY, s = 0.0;
        for (int it = 0; it < max_iter; it++) {
            double sl = 0.0, tl = 0.0;
            const double nb = -beta;
#pragma unroll
            for (int j = 0; j < KPL; j++) {
                if (lane + 32 * j < k) {
                    double e = exp(__dmul_rn(nb, delta[j]));
                    sl = __dadd_rn(sl, e);
                    tl = __dadd_rn(tl, __dmul_rn(e, delta[j]));
                }
            }
            s = warp_sum(sl);
            const double t = warp_sum(tl);
            const double H = __dadd_rn(log(s), __ddiv_rn(__dmul_rn(beta, t), s));
            if (fabs(__dsub_rn(H, ln_u)) <= tol) break;
            if (H > ln_u) {
                lo = beta;
                beta = isinf(hi) ? __dmul_rn(beta, 2.0) : __dmul_rn(0.5, __dadd_rn(lo, hi));
            } else {
                hi = beta;
                beta = __dmul_rn(0.5, __dadd_rn(lo, hi));
            }
        }
        const double nb = -beta;
#pragma unroll
        for (int j = 0; j < KPL; j++) {
            int idx = lane + 32 * j;
            if (idx < k) out[idx] = __ddiv_rn(exp(__dmul_rn(nb, delta[j])), s);
        }
        if (lane == 0) betas[row] = beta;
    }
}

// ---------------------------------------------------------------------------
// Device-wide exclusive scan of a functor-generated sequence (3 kernels).
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256, kScanIPT = 16, kScanTile = kScanThreads * kScanIPT;

template <typename T, typename F>
__global__ void __launch_bounds__(kScanThreads)
k_scan_reduce(F f, int64_t n, T *__restrict__ bsum) {
    __shared__ T s_scan[32];
    __shared__ T s_tot;
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    T acc = 0;
    for (int j = 0; j < kScanIPT; j++) {
        int64_t i = base + (int64_t)j * kScanThreads + threadIdx.x;
        if (i < n) acc += f(i);
    }
    block_exclusive_scan<T>(acc, s_scan, &s_tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = s_tot;
}

template <typename T>
__global__ void __launch_bounds__(1024)
k_scan_mid(T *__restrict__ bsum, int64_t nb, T *__restrict__ total) {
    __shared__ T s_scan[32];
    __shared__ T s_tot;
    __shared__ T s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < nb; b0 += 1024) {
        int64_t b = b0 + threadIdx.x;
        T v = b < nb ? bsum[b] : T(0);
        T x = block_exclusive_scan<T>(v, s_scan, &s_tot);
        if (b < nb) bsum[b] = s_carry + x;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += s_tot;
        __syncthreads();
    }
    if (threadIdx.x == 0 && total) *total = s_carry;
}

template <typename T, typename F>
__global__ void __launch_bounds__(kScanThreads)
k_scan_down(F f, int64_t n, const T *__restrict__ bsum, T *__restrict__ out) {
    __shared__ T s_scan[32];
    __shared__ T s_tot;
    __shared__ T s_carry;
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    if (threadIdx.x == 0) s_carry = bsum[blockIdx.x];
    __syncthreads();
    for (int j = 0; j < kScanIPT; j++) {
        int64_t i = base + (int64_t)j * kScanThreads + threadIdx.x;
        T v = i < n ? f(i) : T(0);
        T x = block_exclusive_scan<T>(v, s_scan, &s_tot);
        if (i < n) out[i] = s_carry + x;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += s_tot;
        __syncthreads();
    }
}

template <typename T, typename F>
static size_t scan_ws(int64_t n) {
    return bh_align(sizeof(T) * bh_blocks(n, kScanTile));
}

template <typename T, typename F>
static int device_scan(F f, int64_t n, T *out, T *total, void *ws,
                       cudaStream_t st) {
    const int nb = bh_blocks(n, kScanTile);
    T *bsum = (T *)ws;
    k_scan_reduce<T, F><<<nb, kScanThreads, 0, st>>>(f, n, bsum);
    k_scan_mid<T><<<1, 1024, 0, st>>>(bsum, nb, total);
    k_scan_down<T, F><<<nb, kScanThreads, 0, st>>>(f, n, bsum, out);
    BH_CHECK_LAUNCH("device_scan");
    return BH_OK;
}

// ---------------------------------------------------------------------------
// Symmetrise: every directed kNN edge e = (i -> j) with conditional c_e
// yields entries (i, j) and (j, i), both carrying c_e.  Sorting the 2NK
// (row * N + col) keys (stable radix sort) groups each (row, col) -- at most
// two entries, one per direction -- in CSR order; the value is
// max((c_a + c_b) / 2N, eps64) cast to float32 (affinity.py:152-153).
// ---------------------------------------------------------------------------
__global__ void k_sym_keys(const int64_t *__restrict__ idx, int64_t n, int64_t k,
                           uint64_t *__restrict__ keys, uint32_t *__restrict__ vals) {
    const int64_t E = n * k;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t i = (uint64_t)(e / k), j = (uint64_t)idx[e];
        keys[e] = i * (uint64_t)n + j;
        keys[E + e] = j * (uint64_t)n + i;
        vals[e] = (uint32_t)e;
        vals[E + e] = (uint32_t)e;
    }
}

struct UniqueFlag {
    const uint64_t *keys;
    __device__ uint32_t operator()(int64_t u) const {
        return (u == 0 || keys[u] != keys[u - 1]) ? 1u : 0u;
    }
};

template <typename V>
__global__ void k_sym_fill(const uint64_t *__restrict__ keys,
                           const uint32_t *__restrict__ vals,
                           const uint32_t *__restrict__ pos, int64_t m,
                           const double *__restrict__ cond, int64_t n,
                           int64_t *__restrict__ row_ptr,
                           int32_t *__restrict__ col, V *__restrict__ val,
                           const int64_t *__restrict__ nnz) {
    const double two_n = 2.0 * (double)n;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < m;
         u += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = keys[u];
        if (u > 0 && keys[u - 1] == key) continue;
        const int64_t o = pos[u];
        double s = cond[vals[u]];
        if (u + 1 < m && keys[u + 1] == key) s = __dadd_rn(s, cond[vals[u + 1]]);
        double p = __ddiv_rn(s, two_n);
        if (p < DBL_EPSILON) p = DBL_EPSILON;
        const int64_t row = (int64_t)(key / (uint64_t)n);
        col[o] = (int32_t)(key % (uint64_t)n);
        val[o] = (V)p;  // .astype(dtype): round to nearest for f32
        // first entry of its row: fill row_ptr for this row and any empty
        // rows before it; the last entry also closes the trailing rows
        const int64_t prev = (o == 0) ? -1 : (int64_t)(keys[u - 1] / (uint64_t)n);
        if (o == 0 || prev != row)
            for (int64_t r = prev + 1; r <= row; r++) row_ptr[r] = o;
        if (o == *nnz - 1)
            for (int64_t r = row + 1; r <= n; r++) row_ptr[r] = *nnz;
    }
}

struct SymLayout {
    size_t keys, vals, skeys, svals, pos, scan, sort, total;
    int64_t m;
    int key_bits;
};

static SymLayout sym_layout(int64_t n, int64_t k) {
    SymLayout L;
    L.m = 2 * n * k;
    int bits = 1;
    while (bits < 64 && ((uint64_t)1 << bits) < (uint64_t)n * (uint64_t)n) bits++;
    // keys are stored as uint64; key_bits > 32 selects the 64-bit sort
    L.key_bits = bits > 32 ? bits : 33;
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += bh_align(b); return o; };
    L.keys = take(8 * L.m);
    L.vals = take(4 * L.m);
    L.skeys = take(8 * L.m);
    L.svals = take(4 * L.m);
    L.pos = take(4 * L.m);
    L.scan = take(scan_ws<uint32_t, UniqueFlag>(L.m));
    L.sort = take(bh_sort_workspace_bytes(L.m, L.key_bits));
    L.total = off;
    return L;
}

// Padded-CSR helpers.
struct PadLen {
    const int64_t *rp;
    __device__ int64_t operator()(int64_t r) const {
        return (rp[r + 1] - rp[r] + 3) & ~(int64_t)3;
    }
};

__global__ void k_pad_finish(const int64_t *__restrict__ rp, int64_t n,
                             int64_t *__restrict__ out_rp,
                             const int64_t *__restrict__ total) {
    if (blockIdx.x == 0 && threadIdx.x == 0) out_rp[n] = *total;
}

template <typename V>
__global__ void k_pad_fill(const int64_t *__restrict__ rp,
                           const int32_t *__restrict__ col,
                           const V *__restrict__ val, int64_t n,
                           const int64_t *__restrict__ orp,
                           int32_t *__restrict__ ocol, V *__restrict__ oval) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = wid; r < n; r += nw) {
        const int64_t s = rp[r], len = rp[r + 1] - s, o = orp[r];
        const int64_t plen = orp[r + 1] - o;
        for (int64_t q = lane; q < plen; q += 32) {
            ocol[o + q] = q < len ? col[s + q] : (int32_t)r;
            oval[o + q] = q < len ? val[s + q] : V(0);
        }
    }
}

}  // namespace bh

using namespace bh;

template <typename S>
static int bsp_impl(const S *sqd, int64_t n, int64_t k, double perplexity,
                    double tol_bits, int64_t max_iter, double *betas,
                    double *cond, bh_stream_t stream) {
    BH_REQUIRE(k >= 1 && k <= 1024, "k must be in [1, 1024] for bh_bsp");
    BH_REQUIRE(perplexity <= (double)k,
               "perplexity exceeds neighborhood size (u=%g, k=%lld)", perplexity,
               (long long)k);
    BH_REQUIRE(perplexity > 1, "perplexity must be > 1, got %g", perplexity);
    BH_REQUIRE(tol_bits > 0, "tolerance must be > 0, got %g", tol_bits);
    if (n == 0) return BH_OK;
    const double ln_u = log(perplexity), tol = tol_bits * log(2.0);
    int grid = bh_blocks(n, 8);
    if (grid > kSMs * 16) grid = kSMs * 16;
    cudaStream_t st = bh_cs(stream);
    const int kpl = (int)((k + 31) / 32);
#define BH_BSP(KPL)                                                           \
    k_bsp<KPL, S><<<grid, 256, 0, st>>>(sqd, n, (int)k, ln_u, tol, (int)max_iter, \
                                     betas, cond)
    if (kpl <= 1) BH_BSP(1);
    else if (kpl <= 2) BH_BSP(2);
    else if (kpl <= 3) BH_BSP(3);
    else if (kpl <= 4) BH_BSP(4);
    else if (kpl <= 8) BH_BSP(8);
    else if (kpl <= 16) BH_BSP(16);
    else BH_BSP(32);
#undef BH_BSP
    BH_CHECK_LAUNCH("k_bsp");
    return BH_OK;
}

extern "C" int bh_bsp(const float *sqd, int64_t n, int64_t k,
                      double perplexity, double tol_bits, int64_t max_iter,
                      double *betas, double *cond, bh_stream_t stream) {
    return bsp_impl(sqd, n, k, perplexity, tol_bits, max_iter, betas, cond,
                    stream);
}

extern "C" int bh_bsp_f64(const double *sqd, int64_t n, int64_t k,
                          double perplexity, double tol_bits, int64_t max_iter,
                          double *betas, double *cond, bh_stream_t stream) {
    return bsp_impl(sqd, n, k, perplexity, tol_bits, max_iter, betas, cond,
                    stream);
}

extern "C" size_t bh_symmetrize_workspace_bytes(int64_t n, int64_t k) {
    return sym_layout(n, k).total;
}

extern "C" int bh_symmetrize_plan(const int64_t *indices, int64_t n, int64_t k,
                                  int64_t *nnz_out, void *ws, size_t ws_bytes,
                                  bh_stream_t stream) {
    BH_REQUIRE(n >= 1 && k >= 1, "empty neighbor graph");
    BH_REQUIRE(2 * n * k < (int64_t)0xFFFFFFFF, "graph too large (2NK >= 2^32)");
    SymLayout L = sym_layout(n, k);
    BH_REQUIRE(ws_bytes >= L.total, "symmetrize workspace too small");
    char *w = (char *)ws;
    cudaStream_t st = bh_cs(stream);
    uint64_t *keys = (uint64_t *)(w + L.keys), *skeys = (uint64_t *)(w + L.skeys);
    uint32_t *vals = (uint32_t *)(w + L.vals), *svals = (uint32_t *)(w + L.svals);
    int grid = bh_blocks(n * k, 256);
    if (grid > kSMs * 32) grid = kSMs * 32;
    k_sym_keys<<<grid, 256, 0, st>>>(indices, n, k, keys, vals);
    BH_CHECK_LAUNCH("k_sym_keys");
    int rc = bh_sort_pairs(keys, vals, L.m, L.key_bits, skeys, svals,
                           w + L.sort, bh_sort_workspace_bytes(L.m, L.key_bits), stream);
    if (rc != BH_OK) return rc;
    // unique-entry positions; the uint32 total is widened into *nnz_out
    uint32_t *pos = (uint32_t *)(w + L.pos);
    uint32_t *tot32 = (uint32_t *)(w + L.keys);  // keys are dead after the sort
    rc = device_scan<uint32_t>(UniqueFlag{skeys}, L.m, pos, tot32, w + L.scan, st);
    if (rc != BH_OK) return rc;
    cudaError_t e = cudaMemsetAsync(nnz_out, 0, sizeof(int64_t), st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(nnz_out, tot32, sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
    return cuda_status(e, "symmetrize nnz");
}

template <typename V>
static int sym_fill_impl(const double *cond, int64_t n, int64_t k,
                         const int64_t *nnz, int64_t *row_ptr, int32_t *col,
                         V *val, void *ws, size_t ws_bytes, bh_stream_t stream) {
    SymLayout L = sym_layout(n, k);
    BH_REQUIRE(ws_bytes >= L.total, "symmetrize workspace too small");
    char *w = (char *)ws;
    int grid = bh_blocks(L.m, 256);
    if (grid > kSMs * 32) grid = kSMs * 32;
    k_sym_fill<V><<<grid, 256, 0, bh_cs(stream)>>>(
        (const uint64_t *)(w + L.skeys), (const uint32_t *)(w + L.svals),
        (const uint32_t *)(w + L.pos), L.m, cond, n, row_ptr, col, val, nnz);
    BH_CHECK_LAUNCH("k_sym_fill");
    return BH_OK;
}

extern "C" int bh_symmetrize_fill(const double *cond, int64_t n, int64_t k,
                                  const int64_t *nnz, int64_t *row_ptr,
                                  int32_t *col, float *val, void *ws,
                                  size_t ws_bytes, bh_stream_t stream) {
    return sym_fill_impl(cond, n, k, nnz, row_ptr, col, val, ws, ws_bytes,
                         stream);
}

extern "C" int bh_symmetrize_fill_f64(const double *cond, int64_t n, int64_t k,
                                      const int64_t *nnz, int64_t *row_ptr,
                                      int32_t *col, double *val, void *ws,
                                      size_t ws_bytes, bh_stream_t stream) {
    return sym_fill_impl(cond, n, k, nnz, row_ptr, col, val, ws, ws_bytes,
                         stream);
}

extern "C" size_t bh_pad_csr_workspace_bytes(int64_t n) {
    return scan_ws<int64_t, PadLen>(n) + 256;
}

extern "C" int bh_pad_csr_size(const int64_t *row_ptr, int64_t n,
                               int64_t *out_row_ptr, int64_t *padded_nnz,
                               void *ws, size_t ws_bytes, bh_stream_t stream) {
    BH_REQUIRE(ws_bytes >= bh_pad_csr_workspace_bytes(n), "pad workspace too small");
    cudaStream_t st = bh_cs(stream);
    int rc = device_scan<int64_t>(PadLen{row_ptr}, n, out_row_ptr, padded_nnz, ws, st);
    if (rc != BH_OK) return rc;
    k_pad_finish<<<1, 32, 0, st>>>(row_ptr, n, out_row_ptr, padded_nnz);
    BH_CHECK_LAUNCH("k_pad_finish");
    return BH_OK;
}

template <typename V>
static int pad_fill_impl(const int64_t *row_ptr, const int32_t *col,
                         const V *val, int64_t n, const int64_t *out_row_ptr,
                         int32_t *out_col, V *out_val, bh_stream_t stream) {
    int grid = bh_blocks(n, 8);
    if (grid > kSMs * 32) grid = kSMs * 32;
    k_pad_fill<V><<<grid, 256, 0, bh_cs(stream)>>>(row_ptr, col, val, n,
                                                   out_row_ptr, out_col, out_val);
    BH_CHECK_LAUNCH("k_pad_fill");
    return BH_OK;
}

extern "C" int bh_pad_csr_fill(const int64_t *row_ptr, const int32_t *col,
                               const float *val, int64_t n,
                               const int64_t *out_row_ptr, int32_t *out_col,
                               float *out_val, bh_stream_t stream) {
    return pad_fill_impl(row_ptr, col, val, n, out_row_ptr, out_col, out_val,
                         stream);
}

extern "C" int bh_pad_csr_fill_f64(const int64_t *row_ptr, const int32_t *col,
                                   const double *val, int64_t n,
                                   const int64_t *out_row_ptr, int32_t *out_col,
                                   double *out_val, bh_stream_t stream) {
    return pad_fill_impl(row_ptr, col, val, n, out_row_ptr, out_col, out_val,
                         stream);
}

// ---------------------------------------------------------------------------
// Morton relabeling of the sparse P (locality of the attractive gathers):
// new row r = old row perm[r]; columns mapped through rank (old -> new).
// Rows keep their padding (pad entries point at their own row).
// ---------------------------------------------------------------------------
namespace bh {

struct PermLen {
    const int64_t *rp;
    const int32_t *perm;
    __device__ int64_t operator()(int64_t r) const {
        const int64_t o = perm[r];
        return rp[o + 1] - rp[o];
    }
};

// 8 lanes per row, 4 rows per warp in flight: rows whose source and
// destination start on a 4-entry boundary and whose length is a multiple
// of 4 (every row of the engine's padded CSR) move as 16-B column / value
// vectors, 4 independent rank gathers per lane; other rows entry by entry.
template <typename V>
__global__ void k_permute_csr_fill(const int64_t *__restrict__ rp,
                                   const int32_t *__restrict__ col,
                                   const V *__restrict__ val,
                                   const int32_t *__restrict__ perm,
                                   const int32_t *__restrict__ rank, int64_t n,
                                   const int64_t *__restrict__ orp,
                                   int32_t *__restrict__ ocol,
                                   V *__restrict__ oval) {
    constexpr int L = 8;  // lanes per row
    const int gl = threadIdx.x & (L - 1);
    const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / L;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / L;
    for (int64_t r = grp; r < n; r += ng) {
        const int64_t o = perm[r], s = rp[o], len = rp[o + 1] - s, d = orp[r];
        if (sizeof(V) == 4 && ((s | d | len) & 3) == 0) {
            for (int64_t q = 4 * gl; q < len; q += 4 * L) {
                const int4 c = *(const int4 *)(col + s + q);
                const float4 v = *(const float4 *)((const float *)val + s + q);
                *(int4 *)(ocol + d + q) =
                    make_int4(rank[c.x], rank[c.y], rank[c.z], rank[c.w]);
                *(float4 *)((float *)oval + d + q) = v;
            }
        } else {
            for (int64_t q = gl; q < len; q += L) {
                ocol[d + q] = rank[col[s + q]];
                oval[d + q] = val[s + q];
            }
        }
    }
}

__global__ void k_set_last(int64_t *__restrict__ out_rp, int64_t n,
                           const int64_t *__restrict__ total) {
    out_rp[n] = *total;
}

}  // namespace bh

extern "C" size_t bh_permute_csr_workspace_bytes(int64_t n) {
    return scan_ws<int64_t, PermLen>(n) + 256;
}

template <typename V>
static int permute_impl(const int64_t *row_ptr, const int32_t *col,
                        const V *val, const int32_t *perm, const int32_t *rank,
                        int64_t n, int64_t *out_row_ptr, int32_t *out_col,
                        V *out_val, void *ws, size_t ws_bytes,
                        bh_stream_t stream) {
    BH_REQUIRE(ws_bytes >= bh_permute_csr_workspace_bytes(n),
               "permute workspace too small");
    cudaStream_t st = bh_cs(stream);
    int64_t *total = (int64_t *)((char *)ws + scan_ws<int64_t, PermLen>(n));
    int rc = device_scan<int64_t>(PermLen{row_ptr, perm}, n, out_row_ptr, total,
                                  ws, st);
    if (rc != BH_OK) return rc;
    k_set_last<<<1, 1, 0, st>>>(out_row_ptr, n, total);
    int grid = bh_blocks(n, 256 / 8);
    if (grid > kSMs * 16) grid = kSMs * 16;
    k_permute_csr_fill<V><<<grid, 256, 0, st>>>(row_ptr, col, val, perm, rank,
                                                n, out_row_ptr, out_col, out_val);
    BH_CHECK_LAUNCH("k_permute_csr_fill");
    return BH_OK;
}

extern "C" int bh_permute_csr(const int64_t *row_ptr, const int32_t *col,
                              const float *val, const int32_t *perm,
                              const int32_t *rank, int64_t n,
                              int64_t *out_row_ptr, int32_t *out_col,
                              float *out_val, void *ws, size_t ws_bytes,
                              bh_stream_t stream) {
    return permute_impl(row_ptr, col, val, perm, rank, n, out_row_ptr, out_col,
                        out_val, ws, ws_bytes, stream);
}

extern "C" int bh_permute_csr_f64(const int64_t *row_ptr, const int32_t *col,
                                  const double *val, const int32_t *perm,
                                  const int32_t *rank, int64_t n,
                                  int64_t *out_row_ptr, int32_t *out_col,
                                  double *out_val, void *ws, size_t ws_bytes,
                                  bh_stream_t stream) {
    return permute_impl(row_ptr, col, val, perm, rank, n, out_row_ptr, out_col,
                        out_val, ws, ws_bytes, stream);
}
