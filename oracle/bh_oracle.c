/*
 * bh_oracle.c -- CPU restatement of the reference Barnes-Hut t-SNE hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * kernels and the CPU baseline that bench.py reports beside them.  Nothing in
 * the product package (paper_2212_11506_b200/) may link, load or call it.
 *
 * Every function restates the algorithm of the reference package `bhtsne`
 * (paths relative to /root/reference/pkg/src/bhtsne/) in plain C with OpenMP,
 * in the reference's f32 run mode: point coordinates, affinities and force
 * outputs are float, every accumulation is double, exactly as the numba
 * kernels upcast (forces.py:60-72, 90-122; quadtree.py:489-508).
 *
 * Parity pin: tests/test_oracle.py checks every function against golden
 * vectors produced by the unmodified reference (tests/golden/make_golden.py),
 * bit-exact for integer work (codes, order, topology, mass) and for the f64
 * results whose operation order is restated exactly (bounds, com, BH forces).
 *
 * Code width.  The reference uses 64-bit Morton codes and MAX_DEPTH = 32
 * (quadtree.py:37,177-185).  The B200 path defaults to 32-bit codes and
 * depth 16; `code_bits` selects either.  In 32-bit mode the quantisation
 * scale is 2^15/r_span, whose code equals the top 32 bits of the reference's
 * 64-bit code, and the tree is the reference builder with
 * MAX_DEPTH = 16 (SURVEY.md 8c ii).
 *
 * Compiled with -ffp-contract=off: the reference's numba kernels contain no
 * FMA contraction, so neither may this restatement.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_STACK_CAP 160 /* forces.py:27 */

static int or_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int or_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
    return omp_get_max_threads();
#else
    (void)t;
    return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* bounds: quadtree.py:133-153                                               */
/* ------------------------------------------------------------------------ */
/* returns 0, or -1 when a coordinate is non-finite (quadtree.py:143-144) */
int or_bounds(const float *y0, const float *y1, int64_t n, double *out3) {
    if (n < 1) return -2;
    float mn0 = y0[0], mx0 = y0[0], mn1 = y1[0], mx1 = y1[0];
    int bad = 0;
    for (int64_t i = 0; i < n; i++) {
        float a = y0[i], b = y1[i];
        if (!isfinite(a) || !isfinite(b)) bad = 1;
        if (a < mn0) mn0 = a;
        if (a > mx0) mx0 = a;
        if (b < mn1) mn1 = b;
        if (b > mx1) mx1 = b;
    }
    if (bad) return -1;
    double dmn0 = mn0, dmx0 = mx0, dmn1 = mn1, dmx1 = mx1;
    double c0 = 0.5 * (dmn0 + dmx0);
    double c1 = 0.5 * (dmn1 + dmx1);
    double h0 = dmx0 - c0, h1 = dmx1 - c1;
    double half = h0 >= h1 ? h0 : h1; /* Python max(): first wins on ties */
    if (half <= 0.0) {
        double m = 1.0;
        if (fabs(c0) > m) m = fabs(c0);
        if (fabs(c1) > m) m = fabs(c1);
        half = 1e-9 * m;
    }
    out3[0] = c0;
    out3[1] = c1;
    out3[2] = half * (1.0 + 1e-12);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Morton codes: quadtree.py:156-185                                         */
/* ------------------------------------------------------------------------ */
static inline uint64_t spread32(uint64_t m) { /* _spread_bits :156-163 */
    m &= 0x00000000FFFFFFFFull;
    m = (m | (m << 16)) & 0x0000FFFF0000FFFFull;
    m = (m | (m << 8)) & 0x00FF00FF00FF00FFull;
    m = (m | (m << 4)) & 0x0F0F0F0F0F0F0F0Full;
    m = (m | (m << 2)) & 0x3333333333333333ull;
    m = (m | (m << 1)) & 0x5555555555555555ull;
    return m;
}

uint64_t or_interleave(uint64_t d0, uint64_t d1) { /* _interleave :166-169 */
    return spread32(d0) | (spread32(d1) << 1);
}

/* code_bits 64: the reference kernel (scale 2^31/r_span, 32 bits per dim).
 * code_bits 32: scale 2^15/r_span, 16 bits per dim (top half of the 64-bit
 * code).  Codes are returned widened to uint64 in both modes. */
void or_morton(const float *y0, const float *y1, int64_t n, double c0,
               double c1, double r_span, int code_bits, uint64_t *codes) {
    double scale = (code_bits == 64 ? 2147483648.0 : 32768.0) / r_span;
    double root0 = c0 - r_span, root1 = c1 - r_span;
    uint64_t mask = code_bits == 64 ? 0xFFFFFFFFull : 0xFFFFull;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        uint64_t m0 = (uint64_t)(((double)y0[i] - root0) * scale);
        uint64_t m1 = (uint64_t)(((double)y1[i] - root1) * scale);
        codes[i] = or_interleave(m0 & mask, m1 & mask);
    }
}

/* stable LSD radix argsort, 8-bit digits over 64 chunks: quadtree.py:188-227 */
void or_radix_argsort(const uint64_t *codes, int64_t n, int code_bits,
                      int64_t *out_order, uint64_t *out_sorted) {
    int64_t nchunks = n >= 64 ? 64 : (n > 0 ? n : 1);
    uint64_t *ka = malloc(sizeof(uint64_t) * (n ? n : 1));
    uint64_t *kb = malloc(sizeof(uint64_t) * (n ? n : 1));
    int64_t *oa = malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t *ob = malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t *hist = calloc((size_t)nchunks * 256, sizeof(int64_t));
    int64_t *offs = calloc((size_t)nchunks * 256, sizeof(int64_t));
    memcpy(ka, codes, sizeof(uint64_t) * n);
    for (int64_t i = 0; i < n; i++) oa[i] = i;
    int passes = code_bits / 8;
    for (int p = 0; p < passes; p++) {
        int shift = 8 * p;
#pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < nchunks; c++) {
            int64_t *h = hist + c * 256;
            memset(h, 0, 256 * sizeof(int64_t));
            int64_t lo = c * n / nchunks, hi = (c + 1) * n / nchunks;
            for (int64_t t = lo; t < hi; t++) h[(ka[t] >> shift) & 0xFF]++;
        }
        int64_t base = 0;
        for (int d = 0; d < 256; d++)
            for (int64_t c = 0; c < nchunks; c++) {
                offs[c * 256 + d] = base;
                base += hist[c * 256 + d];
            }
#pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < nchunks; c++) {
            int64_t local[256];
            memcpy(local, offs + c * 256, sizeof(local));
            int64_t lo = c * n / nchunks, hi = (c + 1) * n / nchunks;
            for (int64_t t = lo; t < hi; t++) {
                int d = (int)((ka[t] >> shift) & 0xFF);
                int64_t pos = local[d]++;
                kb[pos] = ka[t];
                ob[pos] = oa[t];
            }
        }
        uint64_t *tk = ka; ka = kb; kb = tk;
        int64_t *to = oa; oa = ob; ob = to;
    }
    memcpy(out_order, oa, sizeof(int64_t) * n);
    memcpy(out_sorted, ka, sizeof(uint64_t) * n);
    free(ka); free(kb); free(oa); free(ob); free(hist); free(offs);
}

/* ------------------------------------------------------------------------ */
/* Quadtree build: quadtree.py:245-478                                       */
/* ------------------------------------------------------------------------ */
/* The reference builds the canonical level-contiguous tree by splitting each
 * node's sorted-code range on its 2-bit digit with binary searches
 * (_digit_upper_bound :250-259), breadth first.  Its serial top + parallel
 * subtree count/fill phases (:262-396) are a parallel schedule of that same
 * breadth-first construction; the arrays are a pure function of the sorted
 * codes (quadtree.py:19-20).  This restatement runs the breadth-first split
 * level-synchronously (count pass, prefix, fill pass per level, each pass
 * parallel over the level's nodes), which yields the identical arrays. */
typedef struct {
    int64_t n, m, n_levels, cap, max_depth;
    int64_t *level_off; /* n_levels + 1 */
    int64_t *start, *end, *children;
    uint8_t *is_leaf;
    double *center, *radius;
    int64_t *mass;
    float *com;
    double c0, c1, r_span;
} or_tree;

static inline int64_t digit_at(uint64_t code, int depth, int width) {
    return (int64_t)((code >> (width - 2 - 2 * depth)) & 3ull);
}

static inline int64_t digit_upper_bound(const uint64_t *sc, int64_t lo,
                                        int64_t hi, int depth, int width,
                                        int64_t v) {
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (digit_at(sc[mid], depth, width) <= v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

static void tree_reserve(or_tree *t, int64_t need) {
    if (need <= t->cap) return;
    int64_t cap = t->cap ? t->cap : 64;
    while (cap < need) cap *= 2;
    t->start = realloc(t->start, sizeof(int64_t) * cap);
    t->end = realloc(t->end, sizeof(int64_t) * cap);
    t->children = realloc(t->children, sizeof(int64_t) * 4 * cap);
    t->is_leaf = realloc(t->is_leaf, cap);
    t->center = realloc(t->center, sizeof(double) * 2 * cap);
    t->radius = realloc(t->radius, sizeof(double) * cap);
    t->cap = cap;
}

or_tree *or_build_tree(const uint64_t *sc, int64_t n, int code_bits,
                       double c0, double c1, double r_span) {
    or_tree *t = calloc(1, sizeof(or_tree));
    int width = code_bits;
    int D = code_bits / 2; /* MAX_DEPTH: 32 (reference) or 16 */
    t->n = n;
    t->max_depth = D;
    t->c0 = c0; t->c1 = c1; t->r_span = r_span;
    tree_reserve(t, 64);
    t->level_off = malloc(sizeof(int64_t) * (D + 2));
    t->start[0] = 0;
    t->end[0] = n;
    for (int v = 0; v < 4; v++) t->children[v] = -1;
    t->center[0] = c0;
    t->center[1] = c1;
    t->radius[0] = r_span;
    t->level_off[0] = 0;
    t->level_off[1] = 1;
    int64_t lo = 0, hi = 1;
    int depth = 0;
    int64_t *cnt = NULL;
    int64_t cnt_cap = 0;
    for (;;) {
        int64_t width_l = hi - lo;
        if (width_l > cnt_cap) {
            cnt_cap = width_l * 2;
            cnt = realloc(cnt, sizeof(int64_t) * (cnt_cap + 1));
        }
        /* leaf rule (:274-285, :386-387): one point, or at MAX_DEPTH */
#pragma omp parallel for schedule(dynamic, 256)
        for (int64_t k = 0; k < width_l; k++) {
            int64_t nd = lo + k;
            int64_t c = 0;
            int leaf = (t->end[nd] - t->start[nd] == 1) || depth == D;
            t->is_leaf[nd] = (uint8_t)leaf;
            if (!leaf) {
                int64_t prev = t->start[nd];
                for (int v = 0; v < 4; v++) {
                    int64_t e = digit_upper_bound(sc, prev, t->end[nd], depth,
                                                  width, v);
                    if (e > prev) c++;
                    prev = e;
                }
            }
            cnt[k] = c;
        }
        int64_t total = 0;
        for (int64_t k = 0; k < width_l; k++) {
            int64_t c = cnt[k];
            cnt[k] = total;
            total += c;
        }
        if (total == 0) break;
        tree_reserve(t, hi + total);
#pragma omp parallel for schedule(dynamic, 256)
        for (int64_t k = 0; k < width_l; k++) {
            int64_t nd = lo + k;
            if (t->is_leaf[nd]) continue;
            int64_t w = hi + cnt[k];
            double half = t->radius[nd] * 0.5;
            int64_t prev = t->start[nd];
            for (int v = 0; v < 4; v++) {
                int64_t e = digit_upper_bound(sc, prev, t->end[nd], depth,
                                              width, v);
                if (e > prev) {
                    t->start[w] = prev;
                    t->end[w] = e;
                    for (int u = 0; u < 4; u++) t->children[4 * w + u] = -1;
                    t->children[4 * nd + v] = w;
                    t->center[2 * w] = t->center[2 * nd] + ((v & 1) ? half : -half);
                    t->center[2 * w + 1] =
                        t->center[2 * nd + 1] + ((v & 2) ? half : -half);
                    t->radius[w] = half;
                    w++;
                }
                prev = e;
            }
        }
        depth++;
        lo = hi;
        hi = hi + total;
        t->level_off[depth + 1] = hi;
    }
    free(cnt);
    t->m = hi;
    t->n_levels = depth + 1;
    t->mass = calloc(t->m, sizeof(int64_t));
    t->com = calloc(2 * t->m, sizeof(float));
    return t;
}

void or_tree_free(or_tree *t) {
    if (!t) return;
    free(t->level_off); free(t->start); free(t->end); free(t->children);
    free(t->is_leaf); free(t->center); free(t->radius); free(t->mass);
    free(t->com); free(t);
}

void or_tree_dims(const or_tree *t, int64_t *out) {
    out[0] = t->n; out[1] = t->m; out[2] = t->n_levels; out[3] = t->max_depth;
}

void or_tree_copy(const or_tree *t, int64_t *level_off, int64_t *start,
                  int64_t *end, int64_t *children, uint8_t *is_leaf,
                  double *center, double *radius, int64_t *mass, float *com) {
    int64_t m = t->m;
    if (level_off) memcpy(level_off, t->level_off, sizeof(int64_t) * (t->n_levels + 1));
    if (start) memcpy(start, t->start, sizeof(int64_t) * m);
    if (end) memcpy(end, t->end, sizeof(int64_t) * m);
    if (children) memcpy(children, t->children, sizeof(int64_t) * 4 * m);
    if (is_leaf) memcpy(is_leaf, t->is_leaf, m);
    if (center) memcpy(center, t->center, sizeof(double) * 2 * m);
    if (radius) memcpy(radius, t->radius, sizeof(double) * m);
    if (mass) memcpy(mass, t->mass, sizeof(int64_t) * m);
    if (com) memcpy(com, t->com, sizeof(float) * 2 * m);
}

/* ------------------------------------------------------------------------ */
/* summarize: quadtree.py:481-519 (deepest level first, f64 sums, f32 store) */
/* ------------------------------------------------------------------------ */
void or_summarize(or_tree *t, const float *ys0, const float *ys1) {
    for (int64_t level = t->n_levels - 1; level >= 0; level--) {
        int64_t lo = t->level_off[level], hi = t->level_off[level + 1];
#pragma omp parallel for schedule(static)
        for (int64_t nd = lo; nd < hi; nd++) {
            if (t->is_leaf[nd]) {
                int64_t cnt = t->end[nd] - t->start[nd];
                double s0 = 0.0, s1 = 0.0;
                for (int64_t q = t->start[nd]; q < t->end[nd]; q++) {
                    s0 += (double)ys0[q];
                    s1 += (double)ys1[q];
                }
                t->mass[nd] = cnt;
                t->com[2 * nd] = (float)(s0 / (double)cnt);
                t->com[2 * nd + 1] = (float)(s1 / (double)cnt);
            } else {
                int64_t m = 0;
                double a0 = 0.0, a1 = 0.0;
                for (int v = 0; v < 4; v++) {
                    int64_t ch = t->children[4 * nd + v];
                    if (ch >= 0) {
                        int64_t mc = t->mass[ch];
                        m += mc;
                        a0 += (double)mc * (double)t->com[2 * ch];
                        a1 += (double)mc * (double)t->com[2 * ch + 1];
                    }
                }
                t->mass[nd] = m;
                t->com[2 * nd] = (float)(a0 / (double)m);
                t->com[2 * nd + 1] = (float)(a1 / (double)m);
            }
        }
    }
}

/* ------------------------------------------------------------------------ */
/* attractive: forces.py:56-72 (CSR, f64 accumulation, f32 store)            */
/* ------------------------------------------------------------------------ */
void or_attractive(const int64_t *row_off, const int64_t *col,
                   const float *val, const float *y0, const float *y1,
                   int64_t n, float *attr0, float *attr1) {
#pragma omp parallel for schedule(dynamic, 512)
    for (int64_t i = 0; i < n; i++) {
        double yi0 = y0[i], yi1 = y1[i];
        double a0 = 0.0, a1 = 0.0;
        for (int64_t q = row_off[i]; q < row_off[i + 1]; q++) {
            int64_t j = col[q];
            double dx = yi0 - (double)y0[j];
            double dy = yi1 - (double)y1[j];
            double pq = (double)val[q] / (1.0 + dx * dx + dy * dy);
            a0 += pq * dx;
            a1 += pq * dy;
        }
        attr0[i] = (float)a0;
        attr1[i] = (float)a1;
    }
}

/* ------------------------------------------------------------------------ */
/* repulsive Barnes-Hut: forces.py:85-131                                    */
/* ------------------------------------------------------------------------ */
/* counts (optional, 6 per point): internal visits, accepted, leaf-node visits,
 * leaf points touched, max stack depth, leaf-point interactions (no self).
 * These are the SURVEY.md 8(c iii) counters behind the roofline numerator. */
void or_repulsive_bh(const or_tree *t, const int64_t *order, const float *ys0,
                     const float *ys1, const float *y0, const float *y1,
                     int64_t n, double theta, float *rep0, float *rep1,
                     double *zpart, int64_t *counts) {
    double theta2 = theta * theta;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; i++) {
        double yi0 = y0[i], yi1 = y1[i];
        double r0 = 0.0, r1 = 0.0, z = 0.0;
        int64_t stack[OR_STACK_CAP];
        int64_t c_int = 0, c_acc = 0, c_leaf = 0, c_pts = 0, c_max = 1, c_int2 = 0;
        stack[0] = 0;
        int sp = 1;
        while (sp > 0) {
            int64_t nd = stack[--sp];
            if (t->is_leaf[nd]) {
                c_leaf++;
                for (int64_t q = t->start[nd]; q < t->end[nd]; q++) {
                    c_pts++;
                    if (order[q] == i) continue;
                    c_int2++;
                    double dx = yi0 - (double)ys0[q];
                    double dy = yi1 - (double)ys1[q];
                    double k = 1.0 / (1.0 + dx * dx + dy * dy);
                    z += k;
                    r0 += k * k * dx;
                    r1 += k * k * dy;
                }
            } else {
                c_int++;
                double dx = yi0 - (double)t->com[2 * nd];
                double dy = yi1 - (double)t->com[2 * nd + 1];
                double d2 = dx * dx + dy * dy;
                double side = 2.0 * t->radius[nd];
                if (side * side < theta2 * d2) {
                    c_acc++;
                    double k = 1.0 / (1.0 + d2);
                    double mk = (double)t->mass[nd] * k;
                    z += mk;
                    double mk2 = mk * k;
                    r0 += mk2 * dx;
                    r1 += mk2 * dy;
                } else {
                    for (int v = 3; v >= 0; v--) {
                        int64_t ch = t->children[4 * nd + v];
                        if (ch >= 0) stack[sp++] = ch;
                    }
                    if (sp > c_max) c_max = sp;
                }
            }
        }
        rep0[i] = (float)r0;
        rep1[i] = (float)r1;
        zpart[i] = z;
        if (counts) {
            int64_t *c = counts + 6 * i;
            c[0] = c_int; c[1] = c_acc; c[2] = c_leaf; c[3] = c_pts;
            c[4] = c_max; c[5] = c_int2;
        }
    }
}

/* exact O(N^2) repulsion: forces.py:153-173 */
void or_repulsive_exact(const float *y0, const float *y1, int64_t n,
                        float *rep0, float *rep1, double *zpart) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; i++) {
        double yi0 = y0[i], yi1 = y1[i];
        double r0 = 0.0, r1 = 0.0, z = 0.0;
        for (int64_t j = 0; j < n; j++) {
            if (j == i) continue;
            double dx = yi0 - (double)y0[j];
            double dy = yi1 - (double)y1[j];
            double k = 1.0 / (1.0 + dx * dx + dy * dy);
            z += k;
            r0 += k * k * dx;
            r1 += k * k * dy;
        }
        rep0[i] = (float)r0;
        rep1[i] = (float)r1;
        zpart[i] = z;
    }
}

/* ------------------------------------------------------------------------ */
/* perplexity calibration: affinity.py:61-96                                 */
/* ------------------------------------------------------------------------ */
void or_calibrate(const float *sqd, int64_t n, int64_t k, double ln_u,
                  double tol_nats, int64_t max_iter, double *cond,
                  double *betas) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; i++) {
        const float *row = sqd + i * k;
        double *out = cond + i * k;
        double dmax = (double)row[k - 1];
        if (dmax <= 0.0) {
            for (int64_t j = 0; j < k; j++) out[j] = 1.0 / (double)k;
            betas[i] = 1.0;
            continue;
        }
        double dmin = (double)row[0];
        double beta = 1.0, lo = 0.0, hi = INFINITY, s = 0.0;
        for (int64_t it = 0; it < max_iter; it++) {
            s = 0.0;
            double tt = 0.0;
            for (int64_t j = 0; j < k; j++) {
                double delta = (double)row[j] - dmin;
                double e = exp(-beta * delta);
                s += e;
                tt += e * delta;
            }
            double entropy = log(s) + beta * tt / s;
            if (fabs(entropy - ln_u) <= tol_nats) break;
            if (entropy > ln_u) {
                lo = beta;
                beta = isinf(hi) ? beta * 2.0 : 0.5 * (lo + hi);
            } else {
                hi = beta;
                beta = 0.5 * (lo + hi);
            }
        }
        for (int64_t j = 0; j < k; j++)
            out[j] = exp(-beta * ((double)row[j] - dmin)) / s;
        betas[i] = beta;
    }
}

/* ------------------------------------------------------------------------ */
/* KL rows: optimizer.py:227-239                                             */
/* ------------------------------------------------------------------------ */
void or_kl_rows(const int64_t *row_off, const int64_t *col, const float *val,
                const float *y0, const float *y1, int64_t n, double z,
                double *partial) {
#pragma omp parallel for schedule(dynamic, 512)
    for (int64_t i = 0; i < n; i++) {
        double yi0 = y0[i], yi1 = y1[i];
        double acc = 0.0;
        for (int64_t q = row_off[i]; q < row_off[i + 1]; q++) {
            int64_t j = col[q];
            double dx = yi0 - (double)y0[j];
            double dy = yi1 - (double)y1[j];
            double p = (double)val[q];
            acc += p * log(p * z * (1.0 + dx * dx + dy * dy));
        }
        partial[i] = acc;
    }
}

/* ------------------------------------------------------------------------ */
/* momentum / gains update: optimizer.py:161-168, 203-221 (f32 run mode)      */
/* ------------------------------------------------------------------------ */
/* numpy (NEP 50) evaluates `4.0 * (attr - rep / z)` and the gain and velocity
 * expressions in float32 with the Python scalars cast to float32; the mean is
 * a float64 reduction cast back to float32.  Returns -1 - i for the first
 * point with a non-finite gradient (nothing updated), else 0. */
static inline float sgnf(float x) { return (float)((x > 0.0f) - (x < 0.0f)); }

int64_t or_update(float *y0, float *y1, float *v0, float *v1, float *g0,
                  float *g1, const float *attr0, const float *attr1,
                  const float *rep0, const float *rep1, double z, int64_t n,
                  double momentum, double lr, double min_gain) {
    float zf = (float)z, four = 4.0f;
    float mom = (float)momentum, lrf = (float)lr, mg = (float)min_gain;
    float inc = (float)0.2, dec = (float)0.8;
    int64_t bad = -1;
    for (int64_t i = 0; i < n && bad < 0; i++) {
        float a = rep0[i] / zf, b = rep1[i] / zf;
        float gr0 = four * (attr0[i] - a), gr1 = four * (attr1[i] - b);
        if (!isfinite(gr0) || !isfinite(gr1)) bad = i;
    }
    if (bad >= 0) return -1 - bad;
    float *ys[2] = {y0, y1}, *vs[2] = {v0, v1}, *gs[2] = {g0, g1};
    const float *as[2] = {attr0, attr1}, *rs[2] = {rep0, rep1};
    for (int d = 0; d < 2; d++) {
        float *y = ys[d], *v = vs[d], *g = gs[d];
        for (int64_t i = 0; i < n; i++) {
            float q = rs[d][i] / zf;
            float grad = four * (as[d][i] - q);
            int flip = sgnf(grad) != sgnf(v[i]);
            float gn = flip ? g[i] + inc : g[i] * dec;
            if (gn < mg) gn = mg;
            g[i] = gn;
            float t1 = mom * v[i];
            float t2 = lrf * gn;
            float t3 = t2 * grad;
            v[i] = t1 - t3;
            y[i] = y[i] + v[i];
        }
    }
    for (int d = 0; d < 2; d++) {
        float *y = ys[d];
        double s = 0.0;
        for (int64_t i = 0; i < n; i++) s += (double)y[i];
        float m = (float)(s / (double)n);
        for (int64_t i = 0; i < n; i++) y[i] = y[i] - m;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* one full gradient iteration (optimizer.py:171-224) for the CPU baseline   */
/* ------------------------------------------------------------------------ */
/* Runs bounds -> codes -> sort -> tree -> summarize -> attractive ->
 * repulsive -> update, all restated above.  Returns 0, or a negative code on a non-finite input/gradient.
 * stage_s (optional, 5 doubles) receives the wall time of tree, summarize,
 * attractive, repulsive and update, matching StepTimings (optimizer.py:38-39). */
#include <time.h>
static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

int64_t or_gradient_step(float *y0, float *y1, float *v0, float *v1,
                         float *g0, float *g1, const int64_t *row_off,
                         const int64_t *col, const float *val, int64_t n,
                         double theta, double momentum, double lr,
                         double min_gain, int code_bits, double *stage_s) {
    double b[3];
    double t0 = now_s();
    if (or_bounds(y0, y1, n, b) != 0) return -2;
    uint64_t *codes = malloc(sizeof(uint64_t) * n);
    uint64_t *sorted = malloc(sizeof(uint64_t) * n);
    int64_t *order = malloc(sizeof(int64_t) * n);
    or_morton(y0, y1, n, b[0], b[1], b[2], code_bits, codes);
    or_radix_argsort(codes, n, code_bits, order, sorted);
    or_tree *t = or_build_tree(sorted, n, code_bits, b[0], b[1], b[2]);
    float *ys0 = malloc(sizeof(float) * n), *ys1 = malloc(sizeof(float) * n);
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < n; q++) {
        ys0[q] = y0[order[q]];
        ys1[q] = y1[order[q]];
    }
    double t1 = now_s();
    or_summarize(t, ys0, ys1);
    double t2 = now_s();
    float *a0 = malloc(sizeof(float) * n), *a1 = malloc(sizeof(float) * n);
    float *r0 = malloc(sizeof(float) * n), *r1 = malloc(sizeof(float) * n);
    double *zp = malloc(sizeof(double) * n);
    or_attractive(row_off, col, val, y0, y1, n, a0, a1);
    double t3 = now_s();
    or_repulsive_bh(t, order, ys0, ys1, y0, y1, n, theta, r0, r1, zp, NULL);
    double z = 0.0;
    for (int64_t i = 0; i < n; i++) z += zp[i];
    double t4 = now_s();
    int64_t rc = or_update(y0, y1, v0, v1, g0, g1, a0, a1, r0, r1, z, n,
                           momentum, lr, min_gain);
    double t5 = now_s();
    if (stage_s) {
        stage_s[0] = t1 - t0; stage_s[1] = t2 - t1; stage_s[2] = t3 - t2;
        stage_s[3] = t4 - t3; stage_s[4] = t5 - t4;
    }
    or_tree_free(t);
    free(codes); free(sorted); free(order); free(ys0); free(ys1);
    free(a0); free(a1); free(r0); free(r1); free(zp);
    return rc;
}

int or_num_threads(void) { return or_threads(); }
