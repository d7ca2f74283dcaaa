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

// float32 data, register-tiled dot-product filter (the default for bh_knn).
// k_knn_f32 spends one shared-memory operand (a 512-B register write-back)
// per FMA, which caps it at a quarter of the FP32 rate; here a CTA of 128
// threads filters 128 queries x 64 candidates per step as a small GEMM --
// every thread an 8 x 8 tile of dot products, its operands (2 + 2 LDS.128
// per column) reused 8 times.
//
// Filter bound: d^2 = |q|^2 + |s|^2 - 2 q.s.  With the f32 FMA sums nq, ns,
// dot (each within gamma = D 2^-24 / (1 - D 2^-24) of its exact value
// relative to the sum of magnitudes; |q.s| <= (|q|^2 + |s|^2) / 2) the exact
// distance obeys d^2 >= (nq + ns)(1 - 2 gamma - gamma^2) - 2 dot, and the
// three f32 operations evaluating the right-hand side add at most
// 4 * 2^-24 (nq + ns).  kappa = 1e-5 exceeds 2 gamma + gamma^2 + 4 * 2^-24
// for D <= 64, so a candidate with (nq + ns)(1 - kappa) - 2 dot > thr (the
// query's current k-th exact distance, rounded up) cannot enter its list.
// Every other candidate is flagged in the query's 64-bit pass mask; after
// the step the query's owner thread takes them in ascending id order
// through k_knn's exact f64 column-order sum and strict-less insertion, so
// the kept set, the distances and the tie order are k_knn's, bit for bit.
// The filter is weakest (never wrong) for data far from the origin.
#ifndef BH_KNN_TILEQ
#define BH_KNN_TILEQ 128  // queries (= threads) per CTA: 128 or 256
#endif
constexpr int kTileQ = BH_KNN_TILEQ, kTileC = 64;  // CTA tile (queries x candidates)
constexpr int kTileQH = kTileQ / 2;                // a thread's second query quad
constexpr int kTileTQ = kTileQ / 8;                // threads along the queries
constexpr float kKnnKappa = 1e-5f;
constexpr float kKnnKappa64 = 1.1e-5f;  // + the float32 rounding of f64 data

// 4-byte asynchronous global -> shared copy (zero fill when !valid)
__device__ __forceinline__ void cp_async4(float *smem_dst, const float *gsrc,
                                          bool valid) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
    const int sz = valid ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa),
                 "l"(gsrc), "r"(sz)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

template <int DMAX>
struct KnnTileSmem {
    float q[DMAX][kTileQ];       // queries, transposed
    float c[2][kTileC][DMAX + 4];  // candidates (row-major), double-buffered
    float nq[kTileQ], thr[kTileQ], nc[kTileC];
    unsigned mask[kTileQ][2];
};

// KCAP: capacity of the thread-local top-k lists (k <= KCAP); 0 = the lists
// live in caller scratch instead (any k).
// OT = double: float64 data (x64) filtered through its float32 copy x --
// rounding the data moves a distance by at most 4 * 2^-24 (nq + ns), which
// the wider kKnnKappa64 covers -- with the exact sums on the float64 rows.
#ifndef BH_KNN_MINB
#define BH_KNN_MINB (BH_KNN_TILEQ == 128 ? 3 : 2)  // the shared-memory limit; 128-thread CTAs: up to 168 registers
#endif
template <int DMAX, int KCAP, typename OT>
__global__ void __launch_bounds__(kTileQ, BH_KNN_MINB)
k_knn_tile(const float *__restrict__ x, const double *__restrict__ x64,
           int64_t n, int d, int k, int64_t *__restrict__ out_idx,
           OT *__restrict__ out_sqd, double *__restrict__ ws_d,
           int32_t *__restrict__ ws_i) {
    constexpr bool F64 = std::is_same<OT, double>::value;
    extern __shared__ __align__(16) unsigned char knn_smem[];
    KnnTileSmem<DMAX> &S = *reinterpret_cast<KnnTileSmem<DMAX> *>(knn_smem);
    const int tid = threadIdx.x;
    const int64_t q0 = blockIdx.x * (int64_t)kTileQ;
    const int64_t i = q0 + tid;  // the query this thread owns
    const bool ok = i < n;
    // the query tile, transposed (once per CTA), norms and thresholds
    for (int e = tid; e < kTileQ * DMAX; e += kTileQ) {
        const int r = e / DMAX, c = e % DMAX;
        S.q[c][r] = (q0 + r < n && c < d) ? x[(q0 + r) * d + c] : 0.f;
    }
    S.thr[tid] = INFINITY;
    S.mask[tid][0] = S.mask[tid][1] = 0u;
    __syncthreads();
    {
        float a = 0.f;
#pragma unroll
        for (int c = 0; c < DMAX; c++) a = fmaf(S.q[c][tid], S.q[c][tid], a);
        S.nq[tid] = a;
    }
    constexpr bool SCRATCH = KCAP == 0;
    double bd_local[SCRATCH ? 1 : KCAP];
    int32_t bi_local[SCRATCH ? 1 : KCAP];
    double *bd = SCRATCH ? ws_d + (ok ? i : 0) * (int64_t)k : bd_local;
    int32_t *bi = SCRATCH ? ws_i + (ok ? i : 0) * (int64_t)k : bi_local;
    if (ok || !SCRATCH)
        for (int t = 0; t < k; t++) {
            bd[t] = INFINITY;
            bi[t] = -1;
        }
    double thr = INFINITY;
    // this thread's 8 x 8 tile: queries tq4 + {0..3}, 64 + tq4 + {0..3},
    // candidates tc4 + {0..3}, 32 + tc4 + {0..3} (conflict-free LDS.128)
    const int tq4 = (tid % kTileTQ) * 4, tc4 = (tid / kTileTQ) * 4;
    const float om = 1.0f - (F64 ? kKnnKappa64 : kKnnKappa);
    // candidate tiles arrive by cp.async one step ahead of their use
    auto stage = [&](int64_t j0, int buf) {
        // a warp copies whole rows (coalesced reads, conflict-free writes)
        for (int r = tid >> 5; r < kTileC; r += kTileQ / 32) {
            const int64_t j = j0 + r;
#pragma unroll
            for (int c = tid & 31; c < DMAX; c += 32) {
                const bool in = j < n && c < d;
                cp_async4(&S.c[buf][r][c], in ? x + j * d + c : x, in);
            }
        }
        cp_async_commit();
    };
    stage(0, 0);
    int buf = 0;
    for (int64_t j0 = 0; j0 < n; j0 += kTileC, buf ^= 1) {
        cp_async_wait_all();
        __syncthreads();  // this step's tile has landed; the previous step's
                          // owners are done with the other buffer
        if (j0 + kTileC < n) stage(j0 + kTileC, buf ^ 1);
        const float (*Sc)[DMAX + 4] = S.c[buf];
        if (tid < kTileC) {
            float a = 0.f;
#pragma unroll
            for (int c = 0; c < DMAX; c++) a = fmaf(Sc[tid][c], Sc[tid][c], a);
            S.nc[tid] = j0 + tid < n ? a : INFINITY;  // past the end: never passes
        }
        float acc[8][8];
#pragma unroll
        for (int a = 0; a < 8; a++)
#pragma unroll
            for (int b = 0; b < 8; b++) acc[a][b] = 0.f;
#ifndef BH_KNN_UNROLL
#define BH_KNN_UNROLL 7  // 1 / 2 / 4 / 7 / 14 at C3: 6.59 / 6.28 / 5.97 / 5.89 / 6.61 s
#endif
        constexpr int kUnroll = BH_KNN_UNROLL;
#pragma unroll kUnroll
        for (int c = 0; c < DMAX; c += 2) {
            // two columns per round: 8 broadcast LDS.64 of the candidates'
            // rows, 2 + 2 LDS.128 of the transposed queries
            float2 cw[8];
#pragma unroll
            for (int b = 0; b < 8; b++)
                cw[b] = *reinterpret_cast<const float2 *>(
                    &Sc[(b < 4 ? tc4 : 28 + tc4) + b][c]);
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const float4 qa =
                    *reinterpret_cast<const float4 *>(&S.q[c + h][tq4]);
                const float4 qb =
                    *reinterpret_cast<const float4 *>(&S.q[c + h][kTileQH + tq4]);
                const float qv[8] = {qa.x, qa.y, qa.z, qa.w,
                                     qb.x, qb.y, qb.z, qb.w};
#pragma unroll
                for (int a = 0; a < 8; a++)
#pragma unroll
                    for (int b = 0; b < 8; b++)
                        acc[a][b] = fmaf(qv[a], h ? cw[b].y : cw[b].x,
                                         acc[a][b]);
            }
        }
        __syncthreads();  // S.nc is written
        // filter: flag the pairs that may enter
#pragma unroll
        for (int a = 0; a < 8; a++) {
            const int ql = (a < 4 ? tq4 : kTileQH - 4 + tq4) + a;
            const float nqa = S.nq[ql], th = S.thr[ql];
            unsigned m0 = 0u, m1 = 0u;
#pragma unroll
            for (int b = 0; b < 8; b++) {
                const int cl = (b < 4 ? tc4 : 28 + tc4) + b;  // 32 + tc4 + (b - 4)
                const float lower =
                    fmaf(nqa + S.nc[cl], om, -2.0f * acc[a][b]);
                if (!(lower > th)) {
                    if (b < 4) m0 |= 1u << cl;
                    else m1 |= 1u << (cl - 32);
                }
            }
            if (m0) atomicOr(&S.mask[ql][0], m0);
            if (m1) atomicOr(&S.mask[ql][1], m1);
        }
        __syncthreads();
        // the owner inserts its query's flagged candidates, ascending id
        if (ok) {
#pragma unroll 1
            for (int h = 0; h < 2; h++) {
                unsigned m = S.mask[tid][h];
                if (m == 0u) continue;
                S.mask[tid][h] = 0u;
                while (m) {
                    const int r = 32 * h + __ffs(m) - 1;
                    m &= m - 1;
                    const int64_t j = j0 + r;
                    if (j == i || j >= n) continue;
                    // exact: f64, column order, no FMA (knn.py:36-59).
                    // Unrolled over the padded width (the loads and products
                    // overlap; only the ordered sum is a chain): columns past
                    // d are 0 in both tiles and add an exact +0.
                    double e = 0.0;
                    if (F64) {
                        const double *__restrict__ xi = x64 + i * d;
                        const double *__restrict__ xj = x64 + j * d;
#pragma unroll 4
                        for (int c = 0; c < d; c++) {
                            const double diff =
                                __dsub_rn(__ldg(xi + c), __ldg(xj + c));
                            e = __dadd_rn(e, __dmul_rn(diff, diff));
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < DMAX; c++) {
                            const double diff = __dsub_rn((double)S.q[c][tid],
                                                          (double)Sc[r][c]);
                            e = __dadd_rn(e, __dmul_rn(diff, diff));
                        }
                    }
                    if (!(e < thr)) continue;
                    // strict-less insertion: before the first entry > e
                    // (bd[k - 1] > e here), found by bisection; then the
                    // tail moves up one slot, four entries per round trip
                    int lo = 0, hi = k - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (bd[mid] > e) hi = mid;
                        else lo = mid + 1;
                    }
                    const int pos = lo;
                    int t = k - 1;
                    for (; t - 4 >= pos; t -= 4) {
                        const double d0 = bd[t - 1], d1 = bd[t - 2],
                                     d2 = bd[t - 3], d3 = bd[t - 4];
                        const int32_t i0 = bi[t - 1], i1 = bi[t - 2],
                                      i2 = bi[t - 3], i3 = bi[t - 4];
                        bd[t] = d0; bd[t - 1] = d1; bd[t - 2] = d2; bd[t - 3] = d3;
                        bi[t] = i0; bi[t - 1] = i1; bi[t - 2] = i2; bi[t - 3] = i3;
                    }
                    for (; t > pos; t--) {
                        bd[t] = bd[t - 1];
                        bi[t] = bi[t - 1];
                    }
                    bd[pos] = e;
                    bi[pos] = (int32_t)j;
                    thr = bd[k - 1];
                }
            }
            S.thr[tid] = __double2float_ru(__dmul_ru(thr, 1.0 + 1e-6));
        } else {
            S.mask[tid][0] = S.mask[tid][1] = 0u;
        }
    }
    if (ok) {
        for (int t = 0; t < k; t++) {
            out_idx[i * k + t] = bi[t];
            out_sqd[i * k + t] = (OT)bd[t];
        }
    }
}

template <int DMAX, int KCAP, typename OT>
static int knn_tile_launch(const float *x, const double *x64, int64_t n,
                           int d, int k, int64_t *out_idx, OT *out_sqd,
                           double *ws_d, int32_t *ws_i, cudaStream_t st) {
    const size_t smem = sizeof(KnnTileSmem<DMAX>);
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(
            k_knn_tile<DMAX, KCAP, OT>,
            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return cuda_status(e, "k_knn_tile smem");
        attr_set = true;
    }
    k_knn_tile<DMAX, KCAP, OT><<<bh_blocks(n, kTileQ), kTileQ, smem, st>>>(
        x, x64, n, d, k, out_idx, out_sqd, ws_d, ws_i);
    BH_CHECK_LAUNCH("k_knn_tile");
    return BH_OK;
}

// BH_KNN_TILE=0: the per-thread kernels instead of the tile filter (A/B)
static bool knn_tile_filter() {
    static const bool on = [] {
        const char *s = getenv("BH_KNN_TILE");
        return s ? atoi(s) != 0 : true;
    }();
    return on;
}

constexpr int kKnnBigK = 512;  // thread-local lists up to this k

template <int KCAP, typename OT>
static int knn_tile_dispatch(const float *x, const double *x64, int64_t n,
                             int64_t d, int64_t k, int64_t *out_idx,
                             OT *out_sqd, double *ws_d, int32_t *ws_i,
                             cudaStream_t st) {
    const int di = (int)d, ki = (int)k;
#define BH_KNN_TILE_CASE(W)                                                   \
    if (d <= W)                                                               \
        return knn_tile_launch<W, KCAP, OT>(x, x64, n, di, ki, out_idx,       \
                                            out_sqd, ws_d, ws_i, st)
    BH_KNN_TILE_CASE(8);
    BH_KNN_TILE_CASE(16);
    BH_KNN_TILE_CASE(24);
    BH_KNN_TILE_CASE(32);
    BH_KNN_TILE_CASE(40);
    BH_KNN_TILE_CASE(48);
    BH_KNN_TILE_CASE(56);
    BH_KNN_TILE_CASE(64);
#undef BH_KNN_TILE_CASE
    return set_error(BH_ERR_UNSUPPORTED, "the tile filter needs D <= 64");
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

// The tile filter for any k: thread-local lists up to kKnnBigK entries,
// caller scratch beyond.
template <typename OT>
static int knn_tile_any_k(const float *x, const double *x64, int64_t n,
                          int64_t d, int64_t k, int64_t *out_idx, OT *out_sqd,
                          double *wd, int32_t *wi, cudaStream_t st) {
    if (k <= kKnnMaxK)
        return knn_tile_dispatch<kKnnMaxK, OT>(x, x64, n, d, k, out_idx,
                                               out_sqd, wd, wi, st);
    if (k <= kKnnBigK)
        return knn_tile_dispatch<kKnnBigK, OT>(x, x64, n, d, k, out_idx,
                                               out_sqd, wd, wi, st);
    BH_REQUIRE(wd && wi, "k > %d needs the bh_knn_general workspace", kKnnBigK);
    return knn_tile_dispatch<0, OT>(x, x64, n, d, k, out_idx, out_sqd, wd, wi,
                                    st);
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
    if (std::is_same<T, float>::value && d <= 64 && knn_tile_filter()) {
        // any k with narrow rows: the tile filter, its lists thread-local
        // up to kKnnBigK entries and in the scratch beyond
        const float *xf = (const float *)x;
        float *of = (float *)out_sqd;
        return knn_tile_any_k<float>(xf, nullptr, n, d, k, out_idx, of, wd, wi,
                                     bh_cs(stream));
    }
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
        if (knn_tile_filter())
            return knn_tile_dispatch<kKnnMaxK, float>(
                xf, nullptr, n, d, k, out_idx, of, nullptr, nullptr, st);
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

extern "C" int bh_knn_f64_filtered(const double *x, const float *x32,
                                   int64_t n, int64_t d, int64_t k,
                                   int64_t *out_idx, double *out_sqd, void *ws,
                                   size_t ws_bytes, bh_stream_t stream) {
    BH_REQUIRE(x && x32 && out_idx && out_sqd, "null argument");
    BH_REQUIRE(k >= 1 && k <= n - 1, "k must be in [1, %lld], got %lld",
               (long long)(n - 1), (long long)k);
    BH_REQUIRE(d >= 1 && d <= 64,
               "bh_knn_f64_filtered supports 1 <= D <= 64, got %lld",
               (long long)d);
    double *wd = nullptr;
    int32_t *wi = nullptr;
    if (k > kKnnBigK) {
        BH_REQUIRE(ws && ws_bytes >= bh_knn_general_workspace_bytes(n, k),
                   "kNN workspace too small");
        wd = (double *)ws;
        wi = (int32_t *)((char *)ws + bh_align(sizeof(double) * n * k));
    }
    return knn_tile_any_k<double>(x32, x, n, d, k, out_idx, out_sqd, wd, wi,
                                  bh_cs(stream));
}
