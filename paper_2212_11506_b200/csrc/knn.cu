// Exact k-nearest neighbours -- the GPU version of
// knn_exact (knn.py:36-73) with the reference's exact semantics: squared
// distances accumulated in f64 over the columns in order (no FMA), k
// smallest kept by strict-less insertion over ascending candidate ids (ties
// -> lower id), self excluded, distances stored in the data's precision
// (float32 data -> float32 distances; float64 data -> float64, knn.py:72).
//
// One thread per query, its row held in registers as f64; candidate rows are
// staged per CTA in shared memory (f64, broadcast reads).  The partial sum
// is monotone, so a candidate is abandoned as soon as it exceeds the current
// k-th distance.  The per-query top-k lives in thread-local memory.
#include <type_traits>

#include "common.cuh"

namespace bh {

constexpr int kKnnThreads = 128;
constexpr int kKnnTile = 32;
constexpr int kKnnMaxK = 128;

template <int DMAX, typename T>
__global__ void __launch_bounds__(kKnnThreads)
k_knn(const T *__restrict__ x, int64_t n, int d, int k,
      int64_t *__restrict__ out_idx, T *__restrict__ out_sqd) {
    __shared__ double s_c[kKnnTile][DMAX];
    const int64_t i = blockIdx.x * (int64_t)kKnnThreads + threadIdx.x;
    const bool ok = i < n;
    double q[DMAX];
#pragma unroll
    for (int c = 0; c < DMAX; c++) q[c] = (ok && c < d) ? (double)x[i * d + c] : 0.0;
    double bd[kKnnMaxK];
    int32_t bi[kKnnMaxK];
    for (int t = 0; t < k; t++) {
        bd[t] = INFINITY;
        bi[t] = -1;
    }
    double thr = INFINITY;
    for (int64_t j0 = 0; j0 < n; j0 += kKnnTile) {
        __syncthreads();
        for (int e = threadIdx.x; e < kKnnTile * DMAX; e += kKnnThreads) {
            int r = e / DMAX, c = e % DMAX;
            int64_t j = j0 + r;
            s_c[r][c] = (j < n && c < d) ? (double)x[j * d + c] : 0.0;
        }
        __syncthreads();
        if (!ok) continue;
        const int nb = (n - j0) < kKnnTile ? (int)(n - j0) : kKnnTile;
        for (int r = 0; r < nb; r++) {
            const int64_t j = j0 + r;
            if (j == i) continue;
            double acc = 0.0;
            bool keep = true;
#pragma unroll
            for (int c = 0; c < DMAX; c++) {
                if (c < d) {
                    double diff = __dsub_rn(q[c], s_c[r][c]);
                    acc = __dadd_rn(acc, __dmul_rn(diff, diff));
                }
                if ((c & 7) == 7 && acc > thr) {
                    keep = false;
                    break;
                }
            }
            if (!keep || !(acc < thr)) continue;
            int pos = k - 1;
            while (pos > 0 && acc < bd[pos - 1]) {
                bd[pos] = bd[pos - 1];
                bi[pos] = bi[pos - 1];
                pos--;
            }
            bd[pos] = acc;
            bi[pos] = (int32_t)j;
            thr = bd[k - 1];
        }
    }
    if (ok) {
        for (int t = 0; t < k; t++) {
            out_idx[i * k + t] = bi[t];
            out_sqd[i * k + t] = (T)bd[t];
        }
    }
}

// float32 data (bh_knn): the same result as k_knn, with an f32 prefilter.
// Every candidate's distance is first summed in f32 (FMA, early abandon);
// its relative error is below (D + 2) 2^-24 < 4e-6 for D <= 64, so a
// candidate whose f32 distance exceeds the current k-th exact distance by
// the margin 1e-4 cannot enter the list, and only the others get the exact
// f64 column-order sum and the strict-less insertion of k_knn.  The kept
// set, the distances and the tie order are k_knn's, bit for bit; the f32
// pipe does the bulk of the work at twice the f64 rate and with half the
// registers for the query row.
template <int DMAX>
__global__ void __launch_bounds__(kKnnThreads)
k_knn_f32(const float *__restrict__ x, int64_t n, int d, int k,
          int64_t *__restrict__ out_idx, float *__restrict__ out_sqd) {
    __shared__ float s_c[kKnnTile][DMAX];
    // the query rows again for the (rare) exact recompute, padded to stay
    // free of bank conflicts: the registers hold them for the filter only
    __shared__ float s_q[kKnnThreads][DMAX + 1];
    const int64_t i = blockIdx.x * (int64_t)kKnnThreads + threadIdx.x;
    const bool ok = i < n;
    float q[DMAX];
#pragma unroll
    for (int c = 0; c < DMAX; c++) {
        q[c] = (ok && c < d) ? x[i * d + c] : 0.f;
        s_q[threadIdx.x][c] = q[c];
    }
    double bd[kKnnMaxK];
    int32_t bi[kKnnMaxK];
    for (int t = 0; t < k; t++) {
        bd[t] = INFINITY;
        bi[t] = -1;
    }
    double thr = INFINITY;
    float thr32 = INFINITY;
    for (int64_t j0 = 0; j0 < n; j0 += kKnnTile) {
        __syncthreads();
        for (int e = threadIdx.x; e < kKnnTile * DMAX; e += kKnnThreads) {
            const int r = e / DMAX, c = e % DMAX;
            const int64_t j = j0 + r;
            s_c[r][c] = (j < n && c < d) ? x[j * d + c] : 0.f;
        }
        __syncthreads();
        if (!ok) continue;
        const int nb = (n - j0) < kKnnTile ? (int)(n - j0) : kKnnTile;
        for (int r = 0; r < nb; r++) {
            const int64_t j = j0 + r;
            if (j == i) continue;
            float acc = 0.f;
            bool keep = true;
#pragma unroll
            for (int c = 0; c < DMAX; c++) {
                if (c < d) {
                    const float df = q[c] - s_c[r][c];
                    acc = fmaf(df, df, acc);
                }
                if ((c & 7) == 7 && acc > thr32) {
                    keep = false;
                    break;
                }
            }
            if (!keep || acc > thr32) continue;
            // exact: f64, column order, no FMA (knn.py:36-59)
            double e = 0.0;
            for (int c = 0; c < d; c++) {
                const double diff =
                    __dsub_rn((double)s_q[threadIdx.x][c], (double)s_c[r][c]);
                e = __dadd_rn(e, __dmul_rn(diff, diff));
            }
            if (!(e < thr)) continue;
            int pos = k - 1;
            while (pos > 0 && e < bd[pos - 1]) {
                bd[pos] = bd[pos - 1];
                bi[pos] = bi[pos - 1];
                pos--;
            }
            bd[pos] = e;
            bi[pos] = (int32_t)j;
            thr = bd[k - 1];
            thr32 = __double2float_ru(__dmul_ru(thr, 1.0 + 1e-4));
        }
    }
    if (ok) {
        for (int t = 0; t < k; t++) {
            out_idx[i * k + t] = bi[t];
            out_sqd[i * k + t] = (float)bd[t];
        }
    }
}

// Any D, any k (bh_knn_general): the same arithmetic and insertion rule,
// with the query's columns streamed in chunks of kKnnChunk (a tile of 32
// candidate rows per chunk in shared memory, one f64 partial sum per
// candidate in registers) and the running top-k in caller scratch (global,
// L1/L2 resident per thread).  A candidate whose partial sum already
// exceeds the k-th distance after a chunk is dropped from the remaining
// chunks (the sum is monotone).
constexpr int kKnnChunk = 32;

template <typename T>
__global__ void __launch_bounds__(kKnnThreads)
k_knn_general(const T *__restrict__ x, int64_t n, int d, int k,
              int64_t *__restrict__ out_idx, T *__restrict__ out_sqd,
              double *__restrict__ ws_d, int32_t *__restrict__ ws_i) {
    __shared__ double s_c[kKnnTile][kKnnChunk + 1];
    const int64_t i = blockIdx.x * (int64_t)kKnnThreads + threadIdx.x;
    const bool ok = i < n;
    double *bd = ws_d + (ok ? i : 0) * (int64_t)k;
    int32_t *bi = ws_i + (ok ? i : 0) * (int64_t)k;
    if (ok)
        for (int t = 0; t < k; t++) {
            bd[t] = INFINITY;
            bi[t] = -1;
        }
    double thr = INFINITY;
    for (int64_t j0 = 0; j0 < n; j0 += kKnnTile) {
        const int nb = (n - j0) < kKnnTile ? (int)(n - j0) : kKnnTile;
        double acc[kKnnTile];
#pragma unroll
        for (int r = 0; r < kKnnTile; r++) acc[r] = 0.0;
        for (int c0 = 0; c0 < d; c0 += kKnnChunk) {
            const int nc = (d - c0) < kKnnChunk ? d - c0 : kKnnChunk;
            __syncthreads();
            for (int e = threadIdx.x; e < kKnnTile * kKnnChunk; e += kKnnThreads) {
                const int r = e / kKnnChunk, c = e % kKnnChunk;
                const int64_t j = j0 + r;
                s_c[r][c] = (j < n && c < nc) ? (double)x[j * d + c0 + c] : 0.0;
            }
            __syncthreads();
            if (!ok) continue;
            for (int c = 0; c < nc; c++) {
                const double qc = (double)x[i * d + c0 + c];
#pragma unroll
                for (int r = 0; r < kKnnTile; r++) {
                    const double diff = __dsub_rn(qc, s_c[r][c]);
                    acc[r] = __dadd_rn(acc[r], __dmul_rn(diff, diff));
                }
            }
        }
        if (!ok) continue;
        for (int r = 0; r < nb; r++) {
            const int64_t j = j0 + r;
            const double a = acc[r];
            if (j == i || !(a < thr)) continue;
            int pos = k - 1;
            while (pos > 0 && a < bd[pos - 1]) {
                bd[pos] = bd[pos - 1];
                bi[pos] = bi[pos - 1];
                pos--;
            }
            bd[pos] = a;
            bi[pos] = (int32_t)j;
            thr = bd[k - 1];
        }
    }
    if (ok)
        for (int t = 0; t < k; t++) {
            out_idx[i * k + t] = bi[t];
            out_sqd[i * k + t] = (T)bd[t];
        }
}

}  // namespace bh

using namespace bh;

extern "C" size_t bh_knn_general_workspace_bytes(int64_t n, int64_t k) {
    return bh_align(sizeof(double) * n * k) + bh_align(sizeof(int32_t) * n * k);
}

template <typename T>
static int knn_general_impl(const T *x, int64_t n, int64_t d, int64_t k,
                            int64_t *out_idx, T *out_sqd, void *ws,
                            size_t ws_bytes, bh_stream_t stream) {
    BH_REQUIRE(k >= 1 && k <= n - 1, "k must be in [1, %lld], got %lld",
               (long long)(n - 1), (long long)k);
    BH_REQUIRE(d >= 1, "need at least one column");
    BH_REQUIRE(ws_bytes >= bh_knn_general_workspace_bytes(n, k),
               "kNN workspace too small");
    double *wd = (double *)ws;
    int32_t *wi = (int32_t *)((char *)ws + bh_align(sizeof(double) * n * k));
    k_knn_general<T><<<bh_blocks(n, kKnnThreads), kKnnThreads, 0,
                       bh_cs(stream)>>>(x, n, (int)d, (int)k, out_idx,
                                        out_sqd, wd, wi);
    BH_CHECK_LAUNCH("k_knn_general");
    return BH_OK;
}

extern "C" int bh_knn_general(const float *x, int64_t n, int64_t d, int64_t k,
                              int64_t *out_idx, float *out_sqd, void *ws,
                              size_t ws_bytes, bh_stream_t stream) {
    return knn_general_impl(x, n, d, k, out_idx, out_sqd, ws, ws_bytes, stream);
}

extern "C" int bh_knn_general_f64(const double *x, int64_t n, int64_t d,
                                  int64_t k, int64_t *out_idx, double *out_sqd,
                                  void *ws, size_t ws_bytes,
                                  bh_stream_t stream) {
    return knn_general_impl(x, n, d, k, out_idx, out_sqd, ws, ws_bytes, stream);
}

// BH_KNN_F32=0: the f64-only kernel for float32 data as well (A/B)
static bool knn_f32_filter() {
    static const bool on = [] {
        const char *s = getenv("BH_KNN_F32");
        return s ? atoi(s) != 0 : true;
    }();
    return on;
}

template <typename T>
static int knn_impl(const T *x, int64_t n, int64_t d, int64_t k,
                    int64_t *out_idx, T *out_sqd, bh_stream_t stream) {
    BH_REQUIRE(k >= 1 && k <= n - 1, "k must be in [1, %lld], got %lld",
               (long long)(n - 1), (long long)k);
    BH_REQUIRE(k <= kKnnMaxK, "k must be <= %d for bh_knn", kKnnMaxK);
    BH_REQUIRE(d >= 1 && d <= 64, "bh_knn supports 1 <= D <= 64, got %lld",
               (long long)d);
    const int grid = bh_blocks(n, kKnnThreads);
    cudaStream_t st = bh_cs(stream);
    if (std::is_same<T, float>::value && knn_f32_filter()) {
        const float *xf = (const float *)x;
        float *of = (float *)out_sqd;
        // row widths in steps of 8 (the filter's predicated columns issue
        // whether or not they exist)
        if (d <= 16)
            k_knn_f32<16><<<grid, kKnnThreads, 0, st>>>(xf, n, (int)d, (int)k, out_idx, of);
        else if (d <= 24)
            k_knn_f32<24><<<grid, kKnnThreads, 0, st>>>(xf, n, (int)d, (int)k, out_idx, of);
        else if (d <= 32)
            k_knn_f32<32><<<grid, kKnnThreads, 0, st>>>(xf, n, (int)d, (int)k, out_idx, of);
        else if (d <= 40)
            k_knn_f32<40><<<grid, kKnnThreads, 0, st>>>(xf, n, (int)d, (int)k, out_idx, of);
        else if (d <= 48)
            k_knn_f32<48><<<grid, kKnnThreads, 0, st>>>(xf, n, (int)d, (int)k, out_idx, of);
        else if (d <= 56)
            k_knn_f32<56><<<grid, kKnnThreads, 0, st>>>(xf, n, (int)d, (int)k, out_idx, of);
        else
            k_knn_f32<64><<<grid, kKnnThreads, 0, st>>>(xf, n, (int)d, (int)k, out_idx, of);
        BH_CHECK_LAUNCH("k_knn_f32");
        return BH_OK;
    }
    if (d <= 16)
        k_knn<16, T><<<grid, kKnnThreads, 0, st>>>(x, n, (int)d, (int)k, out_idx, out_sqd);
    else if (d <= 32)
        k_knn<32, T><<<grid, kKnnThreads, 0, st>>>(x, n, (int)d, (int)k, out_idx, out_sqd);
    else
        k_knn<64, T><<<grid, kKnnThreads, 0, st>>>(x, n, (int)d, (int)k, out_idx, out_sqd);
    BH_CHECK_LAUNCH("k_knn");
    return BH_OK;
}

extern "C" int bh_knn(const float *x, int64_t n, int64_t d, int64_t k,
                      int64_t *out_idx, float *out_sqd, bh_stream_t stream) {
    return knn_impl(x, n, d, k, out_idx, out_sqd, stream);
}

extern "C" int bh_knn_f64(const double *x, int64_t n, int64_t d, int64_t k,
                          int64_t *out_idx, double *out_sqd, bh_stream_t stream) {
    return knn_impl(x, n, d, k, out_idx, out_sqd, stream);
}
