/*
 * bhtsne_b200.h -- C ABI of the B200-native Barnes-Hut t-SNE hot path.
 *
 * One shared library (paper_2212_11506_b200/libbhtsne_b200.so, sm_100a) that
 * replaces the numba kernels behind the reference package's stage functions
 * (reference: /root/reference/pkg/src/bhtsne/, exported at __init__.py:22-84).
 * Each entry point below names the reference interface it replaces.
 *
 * Conventions
 *  - Every pointer argument is DEVICE memory allocated by the caller (the
 *    Python host uses torch tensors).  The library never allocates, frees or
 *    retains caller memory.
 *  - Scratch comes from the caller: query `bh_*_workspace_bytes`, allocate
 *    that many bytes ZERO-FILLED once, and pass it back on every call.  The
 *    library leaves all counters it keeps there at zero on return, so a
 *    workspace can be reused across calls and CUDA-graph replays.
 *  - Every call is stream-ordered on `stream` (a cudaStream_t; NULL = the
 *    legacy default stream), never synchronises the host, and returns BH_OK
 *    (0) or a negative BH_ERR_* code; `bh_last_error()` (thread-local) then
 *    holds a message.
 *  - Point coordinates are float32 (N, 2) row-major ("(y0, y1)" pairs), the
 *    reference's f32 run mode (io.py:21-30), with f32 pair arithmetic and
 *    float64 accumulation.  The `_f64` twins take float64 coordinates
 *    (and values, forces, velocities, gains) -- the reference's default
 *    f64 run mode -- and compute every pair term in float64 with the
 *    reference's operation order.  Trees carry their precision
 *    (bh_tree_t.precision).
 *  - Morton codes are 32-bit (16 bits per dimension, tree depth <= 16) by
 *    default or 64-bit (the reference's own width, depth <= 32): `code_bits`.
 */
#ifndef BHTSNE_B200_H
#define BHTSNE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BH_ABI_VERSION 1

enum {
    BH_OK = 0,
    BH_ERR_ARG = -1,         /* invalid argument (message in bh_last_error) */
    BH_ERR_CUDA = -2,        /* a CUDA launch/runtime error */
    BH_ERR_CAPACITY = -3,    /* caller buffer too small */
    BH_ERR_UNSUPPORTED = -5, /* e.g. a code width other than 32/64 */
};

typedef void *bh_stream_t; /* cudaStream_t */

/* Bounding square + Morton constants, resident on the device.
 * c0, c1, r_span: compute_bounds (quadtree.py:133-153), computed in f64
 * exactly as the reference.  root0/root1/scale: _morton_kernel's constants
 * (quadtree.py:179-181) for `code_bits`.  shift0/shift1: a pending
 * re-centering (optimizer.py:220-221) that bh_morton applies when asked;
 * bounds already describe the re-centred points.  nonfinite: set to 1 when a
 * coordinate was NaN/Inf (quadtree.py:143-144). */
typedef struct bh_bounds_t {
    double c0, c1, r_span;
    double root0, root1, scale;
    float shift0, shift1;
    int32_t nonfinite;
    int32_t code_bits;
    double shift0_f64, shift1_f64; /* the pending re-centering, f64 mode */
} bh_bounds_t;

/* Optimiser schedule, resident on the device so that whole iterations can be
 * captured in one CUDA graph.  Mirrors TsneConfig (optimizer.py:43-57) and
 * the run() schedule (optimizer.py:316-321): exaggeration applies while
 * iteration < exaggeration_iters, momentum_early while iteration <
 * momentum_switch (MOMENTUM_SWITCH_ITER = 250, optimizer.py:40).
 * `bad` = (iteration << 32 | point) of the first non-finite gradient
 * (optimizer.py:208-211), INT64_MAX while none; `z` = the last Z. */
typedef struct bh_sched_t {
    int32_t iteration;
    int32_t exaggeration_iters;
    int32_t momentum_switch;
    int32_t pad0;
    float exaggeration;
    float momentum_early, momentum_late;
    float learning_rate, min_gain;
    float pad1;
    int64_t bad;
    double z;
    /* the same schedule constants as float64 (the f64 run mode) */
    double exaggeration_f64;
    double momentum_early_f64, momentum_late_f64;
    double learning_rate_f64, min_gain_f64;
} bh_sched_t;

/* The engine's share of the work, resident on the device so
 * that captured CUDA graphs stay valid when bh_partition re-balances it.
 * Storage slots / CSR rows [lo, hi) belong to this rank (lo is a multiple of
 * BH_REP_POINTS_PER_PARTIAL); rows [lo, split) are swept by
 * bh_step_attractive (a side stream, under the tree build), rows
 * [split, hi) inside bh_step_forces.  One GPU: lo = 0, hi = n. */
typedef struct bh_part_t {
    int64_t lo, hi, split;
    int64_t world;
} bh_part_t;

/* Node record of the level-contiguous quadtree (16 bytes):
 *   x, y  : centre of mass (float32, quadtree.py:488-508)
 *   mass  : point count (float32 value; exact below 2^24 points)
 *   info  : bit 31 = leaf; leaf -> bits 0..30 = first point (sorted order);
 *           internal -> bits 0..28 = first child node, bits 29..30 =
 *           (number of children - 1).  Children of a node are consecutive
 *           in the next level, in Morton-digit order (quadtree.py:66-85). */
/* f64 trees (precision 64) use 32-byte records: {x, y} as float64, then
 * {mass, info, 0, 0} as uint32 -- two 16-byte words. */
#define BH_LEAF_BIT 0x80000000u
#define BH_CHILD_MASK 0x1FFFFFFFu
#define BH_NKIDS_SHIFT 29

/* Quadtree arrays (caller-allocated; capacity = n * (max_depth + 1) + 1 is
 * always sufficient, bh_tree_node_bound()).  Replaces MortonQuadtree
 * (quadtree.py:66-85). */
typedef struct bh_tree_t {
    int64_t n_points;
    int64_t node_capacity;
    int32_t code_bits; /* 32 or 64 */
    int32_t max_depth; /* code_bits / 2 */
    float *node;       /* node_capacity records as above (16 or 32 B) */
    int32_t *parent;   /* node_capacity: parent node, -1 for the root */
    int32_t *node_start; /* node_capacity: first point (sorted order) */
    int32_t *leaf_end;   /* node_capacity: one past the last point of each node */
    int32_t *level_off;  /* max_depth + 3 entries: level l = [off[l], off[l+1]),
                            off[max_depth + 2] = number of levels */
    int32_t *order;      /* n: sorted position -> point id */
    void *sorted_codes;  /* n codes (uint32 or uint64) */
    float *ys;           /* 2n: coordinates in sorted order (quadtree.py:476),
                            float32 or float64 per `precision` */
    int32_t *status;     /* device int32: BH_OK or BH_ERR_CAPACITY after build */
    int32_t *rank;       /* optional n: rank[order[t]] = t (NULL: skipped) */
    int32_t precision;   /* 32 (default, also 0) or 64: y/ys/record type */
    int32_t pad;
} bh_tree_t;

const char *bh_last_error(void);
int bh_abi_version(void);
int64_t bh_tree_node_bound(int64_t n, int code_bits);

/* ---- bounds + Morton codes: compute_bounds / morton_codes --------------
 * quadtree.py:133-153, 177-185, 230-242. */
size_t bh_bounds_workspace_bytes(int64_t n);
int bh_bounds(const float *y, int64_t n, int code_bits, bh_bounds_t *out,
              void *ws, size_t ws_bytes, bh_stream_t stream);
/* codes[i] for point i; apply_shift: first re-centre y in place by
 * (shift0, shift1) (the fused update/centering of gradient_step). */
int bh_morton(float *y, int64_t n, const bh_bounds_t *bounds, int code_bits,
              int apply_shift, void *codes, bh_stream_t stream);
/* The engine's tree order: the same quantisation, keyed by the Hilbert
 * index of the cell instead of the Morton interleave.  The top 2d bits still
 * name the depth-d cell, so the canonical tree over these keys has exactly
 * the reference tree's cells and leaves, siblings ordered along the curve;
 * consecutive points are then always neighbours (no Morton jumps), which
 * keeps the traversal's warps coherent.  Not a reference interface. */
int bh_hilbert(float *y, int64_t n, const bh_bounds_t *bounds, int code_bits,
               int apply_shift, void *codes, bh_stream_t stream);
int bh_hilbert_f64(double *y, int64_t n, const bh_bounds_t *bounds,
                   int code_bits, int apply_shift, void *codes,
                   bh_stream_t stream);
int bh_bounds_f64(const double *y, int64_t n, int code_bits, bh_bounds_t *out,
                  void *ws, size_t ws_bytes, bh_stream_t stream);
int bh_morton_f64(double *y, int64_t n, const bh_bounds_t *bounds,
                  int code_bits, int apply_shift, void *codes,
                  bh_stream_t stream);

/* ---- stable radix sort: _radix_argsort (quadtree.py:188-227) ------------
 * Sorts keys (uint32 when key_bits <= 32, else uint64) with ids 0..n-1 as
 * payload, stable, over bits [0, key_bits).  Equivalent to
 * np.argsort(keys, kind="stable") (test_quadtree.py:97-99). */
size_t bh_sort_workspace_bytes(int64_t n, int key_bits);
int bh_sort(const void *keys, int64_t n, int key_bits, void *sorted_keys,
            int32_t *order, void *ws, size_t ws_bytes, bh_stream_t stream);
/* Same, with an explicit uint32 payload (used by the CSR builder). */
int bh_sort_pairs(const void *keys, const uint32_t *vals, int64_t n,
                  int key_bits, void *sorted_keys, uint32_t *sorted_vals,
                  void *ws, size_t ws_bytes, bh_stream_t stream);

/* ---- tree build: build_tree (quadtree.py:399-478) -----------------------
 * Single-pass ballot-scan builder over the sorted codes; bit-identical
 * topology to the reference builder at the same depth.  Also gathers
 * ys = y[order].  On overflow of node_capacity, *tree->status is set to
 * BH_ERR_CAPACITY and the tree is left incomplete. */
size_t bh_tree_workspace_bytes(int64_t n, int code_bits);
int bh_build_tree(const bh_tree_t *tree, const void *y, void *ws,
                  size_t ws_bytes, bh_stream_t stream);
/* y: float32 or float64 (N, 2) per tree->precision. */

/* ---- summarize (quadtree.py:481-519) --------------------------------------
 * Bottom-up centre of mass and count; bit-identical to the reference
 * (f64 sums in reference order, stored in the tree's precision). */
int bh_summarize(const bh_tree_t *tree, void *ws, size_t ws_bytes,
                 bh_stream_t stream);
/* ws: the bh_tree_workspace_bytes() workspace of the build. */

/* Prefix summarize (f32 trees; the engine's per-iteration path): every node
 * is the contiguous run [node_start, leaf_end) of sorted points, so count =
 * end - start and centre = (S[end] - S[start]) / count with S the f64
 * prefix sum of the sorted points -- two launches instead of one per level.
 * Single-point leaves and depth-D buckets are exactly the reference's; an
 * internal centre differs from bh_summarize's child-order f64 sums only by
 * f64 rounding before the f32 store.  ws: the workspace bh_build_tree used
 * (it holds the build's per-tile point sums). */
int bh_summarize_prefix(const bh_tree_t *tree, void *ws, size_t ws_bytes,
                        bh_stream_t stream);

/* ---- attractive force (forces.py:56-82) ---------------------------------
 * attr[i] = sum_t v_t*(y_i - y_j)/(1+|y_i-y_j|^2) over CSR row i, for rows
 * [row_begin, row_end).  v_t is scaled by the exaggeration: `sched` (if not
 * NULL) selects it from the schedule, else `exaggeration` is used.
 * `row_ptr` may be padded (rows start at multiples of 4 entries, pad
 * entries have val 0): set padded=1 to use 128-bit loads. */
int bh_attractive(const int64_t *row_ptr, const int32_t *col,
                  const float *val, int64_t n_rows, int padded,
                  const float *y, int64_t row_begin, int64_t row_end,
                  float exaggeration, const bh_sched_t *sched, float *attr,
                  bh_stream_t stream);

/* ---- repulsive Barnes-Hut force (forces.py:85-150) -----------------------
 * Warp-synchronous traversal over sorted positions [t_begin, t_end) with
 * per-lane acceptance masks (the exact per-point BH semantics of the
 * reference).  Query coordinates: y_query[id] (by point id) or, when NULL,
 * the tree's own ys.  Outputs indexed by point id (sorted_out = 0) or by
 * t - t_begin (sorted_out = 1): rep (float32 pairs), zpart (float64,
 * optional), counts (optional, 4 int32: internal visits, leaf-node visits,
 * leaf points touched, accepted).  zblock (optional; else in ws) receives
 * one f64 partial of Z per 128 consecutive sorted points; z_out (optional)
 * their fixed-order sum (the same reduction bh_sum_partials applies, so Z
 * does not depend on how ranges are split across GPUs). */
size_t bh_repulsive_workspace_bytes(int64_t n);
int bh_repulsive(const bh_tree_t *tree, const bh_bounds_t *bounds,
                 double theta, const float *y_query, int64_t t_begin,
                 int64_t t_end, int sorted_out, float *rep, double *zpart,
                 double *zblock, double *z_out, int32_t *counts, void *ws,
                 size_t ws_bytes, bh_stream_t stream);
/* Both force passes of one iteration in ONE launch (forces.py:56-150 as
 * called by gradient_step, optimizer.py:101-104): bh_attractive over rows
 * [row_begin, row_end) and bh_repulsive over sorted positions
 * [t_begin, t_end) (no query points, zpart or counts), their CTAs
 * interleaved so the issue-bound traversal and the memory-bound CSR sweep
 * share every SM.  Results, including Z, are bitwise those of the two
 * separate calls.  ws: bh_repulsive_workspace_bytes(t_end - t_begin). */
int bh_forces(const bh_tree_t *tree, const bh_bounds_t *bounds, double theta,
              int64_t t_begin, int64_t t_end, int sorted_out, float *rep,
              double *zblock, double *z_out, void *ws, size_t ws_bytes,
              const int64_t *row_ptr, const int32_t *col, const float *val,
              int64_t n_rows, int padded, const float *y, int64_t row_begin,
              int64_t row_end, float exaggeration, const bh_sched_t *sched,
              float *attr, bh_stream_t stream);
/* f64 twins (tree->precision 64): float64 values, coordinates and forces;
 * pair terms in float64 in the reference's operation order, acceptance
 * (2r)^2 < theta^2 d^2 evaluated in float64 as forces.py:112-116. */
int bh_attractive_f64(const int64_t *row_ptr, const int32_t *col,
                      const double *val, int64_t n_rows, int padded,
                      const double *y, int64_t row_begin, int64_t row_end,
                      double exaggeration, const bh_sched_t *sched,
                      double *attr, bh_stream_t stream);
int bh_repulsive_f64(const bh_tree_t *tree, const bh_bounds_t *bounds,
                     double theta, const double *y_query, int64_t t_begin,
                     int64_t t_end, int sorted_out, double *rep, double *zpart,
                     double *zblock, double *z_out, int32_t *counts, void *ws,
                     size_t ws_bytes, bh_stream_t stream);
int bh_forces_f64(const bh_tree_t *tree, const bh_bounds_t *bounds,
                  double theta, int64_t t_begin, int64_t t_end, int sorted_out,
                  double *rep, double *zblock, double *z_out, void *ws,
                  size_t ws_bytes, const int64_t *row_ptr, const int32_t *col,
                  const double *val, int64_t n_rows, int padded,
                  const double *y, int64_t row_begin, int64_t row_end,
                  double exaggeration, const bh_sched_t *sched, double *attr,
                  bh_stream_t stream);
/* *out = fixed-order sum of n per-CTA Z partials (see bh_repulsive). */
int bh_sum_partials(const double *x, int64_t n, double *out,
                    bh_stream_t stream);
#ifndef BH_REP_POINTS_PER_PARTIAL
#define BH_REP_POINTS_PER_PARTIAL 128
#endif

/* ---- exact O(N^2) repulsion (forces.py:153-182) -------------------------- */
size_t bh_repulsive_exact_workspace_bytes(int64_t n);
int bh_repulsive_exact(const float *y, int64_t n, float *rep, double *zpart,
                       double *z_out, void *ws, size_t ws_bytes,
                       bh_stream_t stream);
int bh_repulsive_exact_f64(const double *y, int64_t n, double *rep,
                           double *zpart, double *z_out, void *ws,
                           size_t ws_bytes, bh_stream_t stream);

/* ---- KL divergence rows (optimizer.py:227-239) ---------------------------
 * *kl_out = sum_i sum_t p ln(p Z (1+d^2)) with Z read from *z (device). */
size_t bh_kl_workspace_bytes(int64_t n);
int bh_kl_rows(const int64_t *row_ptr, const int32_t *col, const float *val,
               int64_t n, int padded, const float *y, const double *z,
               double *kl_out, void *ws, size_t ws_bytes, bh_stream_t stream);
int bh_kl_rows_f64(const int64_t *row_ptr, const int32_t *col,
                   const double *val, int64_t n, int padded, const double *y,
                   const double *z, double *kl_out, void *ws, size_t ws_bytes,
                   bh_stream_t stream);

/* ---- momentum / gains update (optimizer.py:161-168, 195-224) -------------
 * grad = 4 (attr - rep / f32(Z)); gains, velocity, y += v, then the mean of
 * the new y is computed (f64) and published, with the bounds of the
 * re-centred points, into *bounds_out (shift0/shift1 = the f32 mean).  The
 * re-centering itself is applied by bh_center or by the next bh_morton
 * (apply_shift=1).  rep is read at rep_rank[i] when rep_rank is not NULL
 * (sorted-order forces of the multi-GPU path), else at i.  Z is sched->z.
 * Increments sched->iteration. */
size_t bh_update_workspace_bytes(int64_t n);
int bh_update(float *y, float *v, float *g, const float *attr,
              const float *rep, const int32_t *rep_rank, int64_t n,
              bh_sched_t *sched,
              bh_bounds_t *bounds_out, int code_bits, void *ws, size_t ws_bytes,
              bh_stream_t stream);
int bh_center(float *y, int64_t n, const bh_bounds_t *bounds,
              bh_stream_t stream);
/* f64 run mode: grad = 4 (attr - rep / Z) with Z in float64, the update in
 * float64 (optimizer.py:161-168 on float64 arrays), shift*_f64 = the f64
 * mean; schedule constants from the *_f64 fields of sched. */
int bh_update_f64(double *y, double *v, double *g, const double *attr,
                  const double *rep, const int32_t *rep_rank, int64_t n,
                  bh_sched_t *sched, bh_bounds_t *bounds_out, int code_bits,
                  void *ws, size_t ws_bytes, bh_stream_t stream);
int bh_center_f64(double *y, int64_t n, const bh_bounds_t *bounds,
                  bh_stream_t stream);

/* ---- the optimiser loop's engine entry points ------------------------------
 * gradient_step (optimizer.py:195-224) and the run() loop (optimizer.py:
 * 316-325) as the engine runs them: points live in "storage slots" (the
 * Morton order of the last relabel), one GPU -- or each of several -- owns
 * the slots and CSR rows of its bh_part_t (device-resident; bh_partition).
 *
 * bh_partition: balanced cuts of [0, n) for `world` GPUs at multiples of
 *   BH_REP_POINTS_PER_PARTIAL (cost of a slot: w_point + its row length),
 *   cuts (world + 1, device int64) and parts[world] (device); rows
 *   [lo, lo + split_frac (hi - lo)) are the side sweep's.  Equal shares when
 *   a balanced range would exceed cap slots.
 * bh_step_attractive: forces.py:56-82 over rows [lo, split) of *part (the
 *   side-stream sweep that overlaps the tree build).
 * bh_step_qlist: the share's slots in the current sorted order (the
 *   entries of tree order[] inside [lo, hi), stable) -- several GPUs only.
 * bh_step_forces: mode 0 = one launch, the traversal of the share's points
 *   in the current Morton order (forces.py:85-150; qlist, or all of
 *   tree->order on one GPU (qlist = NULL); query y[slot], self = its sorted
 *   position rank[slot]; writes rep[slot] and zpart[slot]) interleaved with
 *   the sweep of rows [split, hi); mode 1 = the traversal alone, mode 2 =
 *   the sweep alone (bitwise the same results as mode 0).  ws:
 *   bh_repulsive_workspace_bytes(max_points); max_points bounds hi - lo.
 * bh_step_zsum: zblock[b] = the fixed-order sum of zpart over the share's
 *   128-slot blocks b (the same blocks and sums on any number of GPUs);
 *   z_out (optional, one GPU): their fixed-order total (sched->z).
 * bh_step_update: the update (bh_update) of slots [lo, hi); reduce = 1 (one
 *   GPU, [lo, hi) = [0, n)) also finishes the iteration (mean, bounds of
 *   the re-centred cloud, iteration + 1), else bh_step_finish does that
 *   after the y exchange, bitwise the same.  ysend (optional): the new y of
 *   the share, packed from row 0.
 * bh_pack_rows / bh_unpack_rows: dst[i] = src[lo + i] for the share; and
 *   dst[cuts[r] + j] = gbuf[r * cap + j] (an all-gather of packed shares
 *   with `cap` rows per rank back into slot order). */
int bh_partition(const int64_t *row_ptr, int64_t n, int world, double w_point,
                 double split_frac, int64_t cap, int64_t *cuts,
                 bh_part_t *parts, bh_stream_t stream);
int bh_step_attractive(const int64_t *row_ptr, const int32_t *col,
                       const float *val, int padded, const float *y,
                       const bh_part_t *part, int64_t max_rows,
                       const bh_sched_t *sched, float *attr,
                       bh_stream_t stream);
size_t bh_step_qlist_workspace_bytes(int64_t n);
int bh_step_qlist(const int32_t *order, int64_t n, const bh_part_t *part,
                  int32_t *qlist, void *ws, size_t ws_bytes,
                  bh_stream_t stream);
int bh_step_forces(const bh_tree_t *tree, const bh_bounds_t *bounds,
                   double theta, const float *y, const int32_t *rank,
                   const int32_t *qlist, const bh_part_t *part,
                   int64_t max_points, int mode, float *rep, double *zpart,
                   void *ws, size_t ws_bytes, const int64_t *row_ptr,
                   const int32_t *col, const float *val, int padded,
                   const bh_sched_t *sched, float *attr, bh_stream_t stream);
size_t bh_step_zsum_workspace_bytes(int64_t n);
int bh_step_zsum(const double *zpart, const bh_part_t *part, int64_t n,
                 int64_t max_points, double *zblock, double *z_out, void *ws,
                 size_t ws_bytes, bh_stream_t stream);
int bh_step_update(float *y, float *v, float *g, const float *attr,
                   const float *rep, const bh_part_t *part, int64_t n,
                   bh_sched_t *sched, bh_bounds_t *bounds_out, int code_bits,
                   int reduce, float *ysend, void *ws, size_t ws_bytes,
                   bh_stream_t stream);
int bh_step_finish(const float *y, int64_t n, bh_sched_t *sched,
                   bh_bounds_t *bounds_out, int code_bits, void *ws,
                   size_t ws_bytes, bh_stream_t stream);
int bh_step_attractive_f64(const int64_t *row_ptr, const int32_t *col,
                           const double *val, int padded, const double *y,
                           const bh_part_t *part, int64_t max_rows,
                           const bh_sched_t *sched, double *attr,
                           bh_stream_t stream);
int bh_step_forces_f64(const bh_tree_t *tree, const bh_bounds_t *bounds,
                       double theta, const double *y, const int32_t *rank,
                       const int32_t *qlist, const bh_part_t *part,
                       int64_t max_points, int mode, double *rep,
                       double *zpart, void *ws, size_t ws_bytes,
                       const int64_t *row_ptr, const int32_t *col,
                       const double *val, int padded, const bh_sched_t *sched,
                       double *attr, bh_stream_t stream);
int bh_step_update_f64(double *y, double *v, double *g, const double *attr,
                       const double *rep, const bh_part_t *part, int64_t n,
                       bh_sched_t *sched, bh_bounds_t *bounds_out,
                       int code_bits, int reduce, double *ysend, void *ws,
                       size_t ws_bytes, bh_stream_t stream);
int bh_step_finish_f64(const double *y, int64_t n, bh_sched_t *sched,
                       bh_bounds_t *bounds_out, int code_bits, void *ws,
                       size_t ws_bytes, bh_stream_t stream);
int bh_pack_rows(const void *src, const bh_part_t *part, int64_t cap,
                 int elem_bytes, void *dst, bh_stream_t stream);
int bh_unpack_rows(const void *gbuf, int64_t cap, const int64_t *cuts,
                   int world, int elem_bytes, void *dst, bh_stream_t stream);

/* ---- binary-search perplexity: calibrate_perplexity (affinity.py:61-118) --
 * One warp per row, f64 bisection with the reference's exact schedule. */
int bh_bsp(const float *sqd, int64_t n, int64_t k, double perplexity,
           double tol_bits, int64_t max_iter, double *betas, double *cond,
           bh_stream_t stream);
int bh_bsp_f64(const double *sqd, int64_t n, int64_t k, double perplexity,
               double tol_bits, int64_t max_iter, double *betas, double *cond,
               bh_stream_t stream);

/* ---- symmetrize (affinity.py:121-158) ------------------------------------
 * p_ij = max((p_j|i + p_i|j) / 2N, eps64) as float32 CSR with ascending
 * columns.  Two calls: bh_symmetrize_plan sorts the 2NK directed entries and
 * writes the nnz to *nnz_out (device int64); after the caller allocates the
 * outputs, bh_symmetrize_fill (same workspace, nnz from the plan) writes
 * row_ptr (n+1), col and val (nnz). */
size_t bh_symmetrize_workspace_bytes(int64_t n, int64_t k);
int bh_symmetrize_plan(const int64_t *indices, int64_t n, int64_t k,
                       int64_t *nnz_out, void *ws, size_t ws_bytes,
                       bh_stream_t stream);
int bh_symmetrize_fill(const double *cond, int64_t n, int64_t k,
                       const int64_t *nnz, int64_t *row_ptr, int32_t *col,
                       float *val, void *ws, size_t ws_bytes,
                       bh_stream_t stream);
/* f64 run mode: values stay float64 (no final cast). */
int bh_symmetrize_fill_f64(const double *cond, int64_t n, int64_t k,
                           const int64_t *nnz, int64_t *row_ptr, int32_t *col,
                           double *val, void *ws, size_t ws_bytes,
                           bh_stream_t stream);
/* Pads a CSR so every row starts at a multiple of 4 entries (pad entries:
 * col = row, val = 0).  out_row_ptr has n+1 entries; out capacity from
 * bh_pad_csr_size (device int64 result in *padded_nnz). */
size_t bh_pad_csr_workspace_bytes(int64_t n);
int bh_pad_csr_size(const int64_t *row_ptr, int64_t n, int64_t *out_row_ptr,
                    int64_t *padded_nnz, void *ws, size_t ws_bytes,
                    bh_stream_t stream);
int bh_pad_csr_fill(const int64_t *row_ptr, const int32_t *col,
                    const float *val, int64_t n, const int64_t *out_row_ptr,
                    int32_t *out_col, float *out_val, bh_stream_t stream);
int bh_pad_csr_fill_f64(const int64_t *row_ptr, const int32_t *col,
                        const double *val, int64_t n,
                        const int64_t *out_row_ptr, int32_t *out_col,
                        double *out_val, bh_stream_t stream);

/* ---- relabeling (engine-internal locality; not a reference interface) ----
 * The optimiser periodically renumbers points in the current Morton order so
 * that CSR rows, their column gathers and the traversal's outputs are
 * spatially coherent.  perm[new] = old, rank[old] = new.  Row gathers and
 * scatters move elem_bytes = 4, 8 or 16 bytes per row. */
int bh_gather_rows(const void *src, const int32_t *idx, int64_t n,
                   int elem_bytes, void *dst, bh_stream_t stream);
int bh_scatter_rows(const void *src, const int32_t *idx, int64_t n,
                    int elem_bytes, void *dst, bh_stream_t stream);
int bh_invert_perm(const int32_t *perm, int64_t n, int32_t *inv,
                   bh_stream_t stream);
size_t bh_permute_csr_workspace_bytes(int64_t n);
int bh_permute_csr(const int64_t *row_ptr, const int32_t *col, const float *val,
                   const int32_t *perm, const int32_t *rank, int64_t n,
                   int64_t *out_row_ptr, int32_t *out_col, float *out_val,
                   void *ws, size_t ws_bytes, bh_stream_t stream);
int bh_permute_csr_f64(const int64_t *row_ptr, const int32_t *col,
                       const double *val, const int32_t *perm,
                       const int32_t *rank, int64_t n, int64_t *out_row_ptr,
                       int32_t *out_col, double *out_val, void *ws,
                       size_t ws_bytes, bh_stream_t stream);

/* ---- exact kNN (knn.py:36-73) ---------------------
 * f64 squared distances summed over columns in order, k smallest per row,
 * ties -> lower id, self excluded; distances returned as float32.
 * x: (n, d) float32 row-major, d <= 64, k <= 128. */
int bh_knn(const float *x, int64_t n, int64_t d, int64_t k, int64_t *out_idx,
           float *out_sqd, bh_stream_t stream);
/* Any D and k (the same semantics and results as bh_knn; float32 rows of
 * D <= 64 take bh_knn's tile filter for any k, the rest is slower): the
 * query's columns streamed in chunks, the running top-k in caller scratch of
 * bh_knn_general_workspace_bytes(n, k) bytes. */
size_t bh_knn_general_workspace_bytes(int64_t n, int64_t k);
int bh_knn_general(const float *x, int64_t n, int64_t d, int64_t k,
                   int64_t *out_idx, float *out_sqd, void *ws,
                   size_t ws_bytes, bh_stream_t stream);
int bh_knn_general_f64(const double *x, int64_t n, int64_t d, int64_t k,
                       int64_t *out_idx, double *out_sqd, void *ws,
                       size_t ws_bytes, bh_stream_t stream);
/* f64 run mode: float64 data, distances returned as float64. */
/* float64 data with the float32 tile filter: x32 = x rounded to float32 (the
 * caller's copy); the same results as bh_knn_f64, bit for bit (the filter
 * only drops pairs it proves too far; exact sums on the float64 rows).
 * d <= 64; ws (bh_knn_general_workspace_bytes) only for k > 512, else NULL. */
int bh_knn_f64_filtered(const double *x, const float *x32, int64_t n,
                        int64_t d, int64_t k, int64_t *out_idx,
                        double *out_sqd, void *ws, size_t ws_bytes,
                        bh_stream_t stream);
int bh_knn_f64(const double *x, int64_t n, int64_t d, int64_t k,
               int64_t *out_idx, double *out_sqd, bh_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* BHTSNE_B200_H */
