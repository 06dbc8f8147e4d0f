/*
 * lts_sm100.h -- C ABI of the B200 (sm_100a) Localized Topological
 * Simplification hot path (liblts_sm100.so).
 *
 * The reference (arXiv 2009.00083, /root/reference/pkg) is a Python/numba
 * package whose operator boundary is a set of flat-array kernels
 * (_kernels.py:1-9) behind the Python types of order.py / critical.py and the
 * SPEC engine.  Each entry point below replaces one of those
 * interfaces; the replaced reference interface is cited next to it.
 *
 * Conventions
 *  - Grids are regular 2D/3D Freudenthal grids, dims = (nx, ny[, nz]),
 *    vertex ids x-fastest (reference triangulation.py:8).  n = prod(dims).
 *  - Every pointer marked "device" is CUDA device memory; the caller owns all
 *    buffers, including the workspace (lts_workspace_size).  No allocation
 *    happens inside a call.  Work is ordered on `stream` (a cudaStream_t, or
 *    NULL for the legacy default stream).  Calls that return a data-dependent
 *    status synchronise `stream` before returning.
 *  - Ranks and vertex ids are int32 on the device (n < 2^31).
 *  - Return value: LTS_OK (0) or one of the LTS_E* codes below;
 *    lts_last_error() gives a message.
 */
#ifndef LTS_SM100_H
#define LTS_SM100_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LTS_OK 0
#define LTS_E_FIELD_NONFINITE 1      /* order.py:35-36 FieldError            */
#define LTS_E_BAD_DIMS 2             /* triangulation.py:133-136 MeshError   */
#define LTS_E_CONSTRAINT_NOT_EXTREMUM 3 /* SPEC.md:353 ConstraintNotExtremum */
#define LTS_E_LOCALIZE_NO_MIN 4      /* _kernels.py:479-480 status 1         */
#define LTS_E_VERIFY_FAILED_AT_CAP 5 /* SPEC.md:388 outer loop exhausted     */
#define LTS_E_WORKSPACE 6            /* workspace too small                  */
#define LTS_E_CUDA 7                 /* CUDA runtime error                   */
#define LTS_E_NO_SADDLE 8            /* every maximum discarded: no saddle   */
#define LTS_E_INVALID 9              /* invalid argument                     */

#define LTS_MAX_REPORT_PASSES 64
#define LTS_NUM_PHASES 12

/* phase indices of lts_report_t.phase_ms */
#define LTS_PH_ORDER 0      /* A1/A2: finiteness + radix sort + rank scatter  */
#define LTS_PH_CLASSIFY 1   /* A3: stencil classification (all calls)        */
#define LTS_PH_DISCOVER 2   /* A6: ascent forest, Boruvka saddles, regions   */
#define LTS_PH_ASSEMBLE 3   /* A7: region lists by ascending rank            */
#define LTS_PH_LOCALIZE 4   /* A8: alternating priority floods               */
#define LTS_PH_INTEGRATE 5  /* A9: prefix-count order integration            */
#define LTS_PH_REALIZE 6    /* A13: saddle-value gathers                     */
#define LTS_PH_VERIFY 7     /* A11/A12: restore + verify                     */
#define LTS_PH_TOTAL 8
#define LTS_PH_FLOOD_KERNEL 9    /* device time of the large-region flood kernel  */
#define LTS_PH_FLOOD_LAUNCHES 10 /* its launch count (a count, not ms)           */
#define LTS_PH_FLOOD_SLOTS 11    /* region slots it flooded, summed over launches */

typedef struct {
  int32_t max_iterations;           /* SPEC.md:303 maxIterations (default 100)  */
  int32_t restore_interior_extrema; /* SPEC.md:302 (default 1)                  */
  int32_t collect_timing;           /* record CUDA-event phase times            */
  int32_t reserved0;
  /* SPEC.md:306-309 per-region N_I: when non-NULL (device int32), every
   * pass appends the N_I of each of its regions (region order of that pass,
   * passes in execution order) while fewer than region_ni_capacity entries
   * are written; lts_report_t.region_ni_count gives the total.               */
  int32_t *region_ni_out;
  int64_t region_ni_capacity;
  int32_t reserved[4];
} lts_options_t;

typedef struct {
  int32_t kind;        /* 0 maxima pass, 1 minima pass                         */
  int32_t n_iter_max;  /* max N_I over regions                                 */
  int64_t seeds;       /* discarded extrema (propagation seeds)                */
  int64_t regions;
  int64_t claimed;     /* vertices flattened in this pass                      */
  int64_t largest;     /* largest region size, saddle included                 */
  int64_t capped;      /* regions that hit the iteration cap (status 2)        */
  int64_t shared_saddles; /* regions whose saddle is shared with a sibling     */
  int64_t maxima_edges;   /* edges of the maxima graph (discover)              */
  int32_t boruvka_rounds; /* Boruvka rounds to settle every saddle level       */
  int32_t big_regions;    /* regions handled by the CTA flood kernel           */
} lts_pass_report_t;

typedef struct {
  int32_t ok;                /* verify_constraints passed                      */
  int32_t outer_iterations;  /* executed outer iterations                      */
  int32_t restored;          /* restored preserved extrema                     */
  int32_t n_passes;
  int64_t extra_max, lost_max, extra_min, lost_min; /* final verify counts     */
  int64_t region_ni_count;   /* per-region N_I entries produced (all passes)   */
  lts_pass_report_t passes[LTS_MAX_REPORT_PASSES];
  double phase_ms[LTS_NUM_PHASES];
} lts_report_t;

/* Device views into the workspace describing the regions of the most recent
 * pass run by lts_remove_pass (valid until the next call on that workspace). */
typedef struct {
  int64_t regions;            /* R                                             */
  int64_t slots;              /* sum of region sizes incl. saddles             */
  const int64_t *region_ptr;  /* device, R+1                                   */
  const int32_t *region_verts;/* device, slots: [saddle, ascending-rank verts] */
  const int32_t *local_rank;  /* device, slots: final local order (s = k-1)    */
  const int32_t *n_iters;     /* device, R                                     */
  const int32_t *status;      /* device, R: 0 ok, 2 capped                     */
  const int32_t *topseed;     /* device, R: max effective rank in the region   */
} lts_regions_view_t;

/* library identity */
const char *lts_version(void);
const char *lts_last_error(void);

/* Workspace bytes needed for grids of these dims. */
int lts_workspace_size(int ndim, const int64_t *dims, size_t *bytes);

/* Order field F: replaces compute_order_field (order.py:86-91) and the
 * finiteness check of ScalarField (order.py:30-36).  Stable by (value, id);
 * -0.0 == +0.0.  f, rank, inverse: device, n.  inverse may be NULL.
 * ndim 1 with dims = {n}: the vertices of an explicit mesh.
 * Returns LTS_E_FIELD_NONFINITE on NaN/inf (synchronises stream). */
int lts_order_field(const float *f, int ndim, const int64_t *dims, int32_t *rank,
                    int32_t *inverse, void *ws, size_t ws_bytes, void *stream);

/* ScalarField finiteness (reference order.py:35-36): LTS_E_FIELD_NONFINITE
 * if f (device float32, n) holds a NaN or +-inf, else LTS_OK.  Synchronous. */
int lts_check_field(const float *f, int64_t n, void *stream);

/* Literal numeric realization: replaces realize_numeric / realize_sweep
 * (order.py:102-116, _kernels.py:84-99) in float64.  g (device float64, n)
 * holds f on entry and is lowered in place along the descending order of
 * `inverse` (device int32, n): a vertex violating the order under (value, id)
 * tie-breaking takes g[prev] - zeta, or nextafter(g[prev], -inf) when that
 * does not decrease.  The sweep is sequential by definition; it runs on one
 * CTA that stages the gathered values through shared memory. */
int lts_realize_numeric(double *g, const int32_t *inverse, int64_t n, double zeta, void *stream);

/* Classification: replaces classify_all / classify_grid (critical.py:95-112,
 * _kernels.py:128-156).  rank: device int32 n.  flags (device uint8 n, may be
 * NULL): bit0 minimum (lower==0), bit1 maximum (upper==0).  lower/upper
 * (device int16 n, may be NULL): link component counts with the reference's
 * link-pair tables (triangulation.py:52-78). */
int lts_classify(const int32_t *rank, int ndim, const int64_t *dims, uint8_t *flags,
                 int16_t *lower, int16_t *upper, void *stream);

/* One removal pass: discover_regions -> localize_simplify_region ->
 * integrate_local_orders (_kernels.py:194-303, 578-591).
 * kind 0: maxima pass on rank; kind 1: minima pass (maxima machinery on the
 * reversed order, order.py:54-56).  Seeds are the extrema of `rank` of that
 * kind that are not marked in pmark (device uint8 n; bit0 preserved minimum,
 * bit1 preserved maximum).  rank/inverse in, new_rank/new_inverse out (device
 * int32 n; may not alias the inputs).  g (device float32 n, may be NULL) is
 * flattened in place: every claimed vertex takes its region saddle's value
 * (contract D1).  view (host, may be NULL) receives the region data. */
int lts_remove_pass(int kind, const int32_t *rank, const int32_t *inverse, const uint8_t *pmark,
                    int ndim, const int64_t *dims, int32_t max_iterations, int32_t *new_rank,
                    int32_t *new_inverse, float *g, lts_pass_report_t *rep,
                    lts_regions_view_t *view, void *ws, size_t ws_bytes, void *stream);

/* Full LTS pass: replaces SPEC simplify_field =
 * order field -> classify -> {maxima pass, minima pass, restore, verify}*
 * -> numeric realization (contract D1).  f: device float32 n.  pres_max /
 * pres_min: device int64 vertex ids (may be empty; the global extremum is
 * added).  order (device int32 n) may be NULL, else it is
 * used as F instead of sorting f.  Outputs g (device float32 n) and G (device
 * int32 n, the final order's ranks).  rep/opt are host structs (opt may be
 * NULL for defaults).  f and g may both be NULL when order is given
 * (remove_extrema: orders only, no numeric realization). */
int lts_simplify(const float *f, int ndim, const int64_t *dims, const int64_t *pres_max,
                 int64_t n_max, const int64_t *pres_min, int64_t n_min, const int32_t *order,
                 float *g, int32_t *G, lts_report_t *rep, const lts_options_t *opt, void *ws,
                 size_t ws_bytes, void *stream);

/* Extremum-saddle pairs of the persistence-driven mode (reference
 * pairs_sweep, _kernels.py:309-421): kind 0 pairs every
 * maximum, kind 1 every minimum (reversed order, negated values).  Outputs,
 * each of n entries (the first *count_out used): extrema_out = extremum vertex
 * ids ascending, saddle_out = the junction vertex each one dies at when its
 * persistence |f(extremum) - f(saddle)| (float64) is below epsilon, else -1
 * (survivor, including the global extremum).  order may be NULL (computed
 * from f).  Synchronous on the stream (returns after the pairs are written). */
int lts_extremum_pairs(const float *f, const int32_t *order, int ndim, const int64_t *dims, int kind,
                       double epsilon, int32_t *extrema_out, int32_t *saddle_out, int64_t *count_out, void *ws,
                       size_t ws_bytes, void *stream);

/* ---- explicit triangle meshes ---------------------------
 * The reference's explicit 2-manifold meshes (build_explicit_triangulation,
 * triangulation.py:172-250) reach its kernels as a symmetric CSR adjacency
 * indptr[n+1] / indices[nnz] plus per-vertex link edges (link_ptr[n+1],
 * link_a / link_b: the two other vertices of every triangle of the vertex).
 * The device path takes the same arrays (device int32).  Vertex degrees must
 * be <= 16 (LTS_E_BAD_DIMS otherwise).  lts_order_field covers explicit meshes
 * with ndim = 1, dims = {n}. */

/* Workspace bytes for an explicit mesh of n vertices. */
int lts_workspace_size_csr(int64_t n, size_t *bytes);

/* classify_all on an explicit mesh: replaces classify_explicit
 * (_kernels.py:159-187).  flags / lower / upper as lts_classify; the link
 * arrays are needed only for the counts (may be NULL with lower/upper NULL). */
int lts_classify_csr(const int32_t *rank, int64_t n, const int32_t *indptr, const int32_t *indices,
                     const int32_t *link_ptr, const int32_t *link_a, const int32_t *link_b, uint8_t *flags,
                     int16_t *lower, int16_t *upper, void *stream);

/* lts_remove_pass on an explicit mesh (discover_sweep / localize_regions over
 * the CSR, _kernels.py:194-303, 578-591). */
int lts_remove_pass_csr(int kind, const int32_t *rank, const int32_t *inverse, const uint8_t *pmark, int64_t n,
                        const int32_t *indptr, const int32_t *indices, int32_t max_iterations, int32_t *new_rank,
                        int32_t *new_inverse, float *g, lts_pass_report_t *rep, lts_regions_view_t *view, void *ws,
                        size_t ws_bytes, void *stream);

/* lts_simplify with HOST buffers, the form the reference's numpy-facing
 * simplify_field binds directly: f_host (float32 n), the
 * preserve lists (int64) and the outputs g_host (float32 n) / G_host (int32 n)
 * are host memory (page-locked for asynchronous copies).  dev: device scratch
 * of lts_host_scratch_size bytes (f, g and the lists on the device).  The
 * copy of g to the host is queued as soon as the last pass has realised it,
 * beside that pass's floods; the call returns with both outputs complete. */
int lts_host_scratch_size(int ndim, const int64_t *dims, int64_t n_max, int64_t n_min, size_t *bytes);
int lts_simplify_host(const float *f_host, int ndim, const int64_t *dims, const int64_t *pres_max_host,
                      int64_t n_max, const int64_t *pres_min_host, int64_t n_min, float *g_host,
                      int32_t *G_host, lts_report_t *rep, const lts_options_t *opt, void *dev,
                      size_t dev_bytes, void *ws, size_t ws_bytes, void *stream);

/* lts_simplify on an explicit mesh (SPEC.md:348-356 over any triangulation). */
int lts_simplify_csr(const float *f, int64_t n, const int32_t *indptr, const int32_t *indices,
                     const int64_t *pres_max, int64_t n_max, const int64_t *pres_min, int64_t n_min,
                     const int32_t *order, float *g, int32_t *G, lts_report_t *rep, const lts_options_t *opt,
                     void *ws, size_t ws_bytes, void *stream);

/* Roofline micro-benchmarks (diagnostics): L2 flushed before each rep, CUDA
 * events around the kernel(s) only.  out_ms (host, 4): [0] order-field sort,
 * [1] classification (flags), [2] classification + ascent pointer, [3] 0. */
int lts_bench_kernels(const float *f, int ndim, const int64_t *dims, int reps, double *out_ms,
                      void *ws, size_t ws_bytes, void *stream);

/* Diagnostics: enable (1) / read per-region counters of the large-region
 * flood kernel: out[i*24 + (k, steps, candidates, committed, flood cycles,
 * check cycles, init cycles, n_iters, per-phase cycles 8..14, climb
 * extractions, gather chunk iterations, gather scan / extract cycles, climb
 * steps)] for the first nregions (<= 256) big regions. */
int lts_debug_big_stats(int enable, int64_t *out, int nregions);

/* Number of CUDA kernels this library launched since load (diagnostics). */
int64_t lts_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* LTS_SM100_H */
