/*
 * cqk_b200.h -- C-ABI of the B200-native CQK / simplex / l1 solver.
 *
 * Drop-in boundary for the reference package `cqksolve` (a pure-Python
 * package; its "operator API" is the Python function surface re-exported in
 * cqksolve/__init__.py:3-49).  Each entry point below names the reference
 * function it replaces.  Plain pointers and sizes only; `mem` says whether the
 * array pointers are host memory (the library stages them through HBM and
 * copies results back) or device memory (zero-copy).
 *
 * Status codes mirror the reference's outcomes and exceptions:
 *   CQK_SOLVED / CQK_INFEASIBLE      -> Status.SOLVED / Status.INFEASIBLE
 *                                       (newton.py:33-35)
 *   CQK_E_DOMAIN (+field, index)     -> DomainError(field, index)  (core.py:30-36)
 *   CQK_E_MAXITER                    -> MaxIterationsError          (newton.py:42-49)
 *   CQK_E_CONTRACT                   -> ContractViolation           (newton.py:38-39)
 *   CQK_E_EMPTY                      -> EmptyIndexSet               (simplex.py:33-34)
 *   CQK_E_CUDA / CQK_E_ARG / CQK_E_TIMEOUT -> library errors (cqk_last_error())
 */
#ifndef CQK_B200_H
#define CQK_B200_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define CQK_ABI_VERSION 1

enum {
  CQK_SOLVED = 0,
  CQK_INFEASIBLE = 1,
  CQK_E_DOMAIN = -1,
  CQK_E_MAXITER = -2,
  CQK_E_CONTRACT = -3,
  CQK_E_CUDA = -4,
  CQK_E_ARG = -5,
  CQK_E_EMPTY = -6,
  CQK_E_TIMEOUT = -7,
  CQK_SPARSE_DENSE = 2,     /* spx_project_sparse_f64: take the dense route */
  CQK_SPARSE_OVERFLOW = 3,  /* ... more than cap nonzero entries (count set) */
};

/* DomainError.field codes */
enum { CQK_F_D = 0, CQK_F_A, CQK_F_B, CQK_F_L, CQK_F_U, CQK_F_R, CQK_F_BOUNDS, CQK_F_Y,
       CQK_F_XBAR };

enum { CQK_MEM_HOST = 0, CQK_MEM_DEVICE = 1 };

/* Decision-logic variant: which reference driver's control flow to replay. */
enum {
  CQK_VARIANT_SOLVE = 0,  /* newton.solve_cqk            newton.py:209-342  */
  CQK_VARIANT_JACOBI = 1, /* parallel.jacobi_solve       parallel.py:371-500 */
  CQK_VARIANT_PAR = 2,    /* parallel.par_solve_cqk      parallel.py:174-327 */
};

/* SolverOptions (newton.py:52-67) plus device knobs. */
typedef struct {
  int32_t variable_fixing;  /* SolverOptions.variable_fixing (ignored by JACOBI) */
  int32_t max_iterations;   /* SolverOptions.max_iterations */
  double tolerance_scale;   /* <= 0 or NaN: eps(dtype)^(3/4) */
  int32_t variant;          /* CQK_VARIANT_* */
  int32_t check;            /* run validate() first (check=True) */
  double lambda0;           /* NaN: the reference initializer; else explicit start */
  double compact_ratio;     /* physical compaction when fixed/present >= ratio;
                               NaN = default 0.25, >1 = never */
  int32_t record_trace;     /* keep (lam, phi, dminus, dplus) per phi evaluation */
  int32_t simplex_start;    /* simplex / l1 start when lambda0 is NaN: 0 = (r - sum y)/n,
                               1 = min((r - sum y)/n, r - max y) (both upper bounds;
                               the reference's `lambda0=` route, simplex.py:246-250),
                               2 = chunked Algorithm 2 (simplex.py:243-245 route with
                               par_simplex_init, parallel.py:330-368) */
} cqk_options;

/* SolveOutcome (newton.py:93-103) plus measurement counters. */
typedef struct {
  int32_t status;
  int32_t domain_field;
  int64_t domain_index;     /* -1: not element specific */
  double lam;               /* multiplier (NaN when infeasible) */
  double lam0;              /* initial multiplier actually used */
  int64_t iterations;
  int64_t phi_evals;
  int64_t fixed_count;
  double bracket_lo, bracket_hi;
  int64_t elems_read;       /* element-passes streamed (x bytes/elem = bytes) */
  int64_t elems_written;    /* element writes (compaction + outputs) */
  int64_t bytes_model;      /* algorithmic HBM bytes of the whole solve */
  double device_ms;         /* kernel time, CUDA events on the solve stream */
  int32_t launches;         /* kernels launched by this call */
  int32_t trace_len;        /* rows available via cqk_get_trace */
} cqk_result;

typedef struct cqk_handle cqk_handle;

/* Library / handle management ------------------------------------------------ */
int cqk_abi_version(void);
const char *cqk_last_error(void);
/* Create a handle bound to CUDA device `device`; owns a stream, scratch and the
   persistent-kernel state.  A handle is not re-entrant. */
int cqk_create(cqk_handle **out, int device);
int cqk_destroy(cqk_handle *h);
/* Run subsequent work on `stream` (cudaStream_t; cudaStreamLegacy = 0x1 is
   accepted); NULL = the handle's own non-blocking stream. */
int cqk_set_stream(cqk_handle *h, void *stream);
int cqk_device_info(cqk_handle *h, int32_t *sm_count, int32_t *ctas, int32_t *threads);
/* Per-pass device timeline of the last persistent solve: rows of 20 int64
   {phase, elements streamed, compacted, t_decide, t_all_arrived, t_released,
   t_cta1_arrived, t_cta1_woke, last_cta, t_last_arrived, then for the TMA CQK kernel
   CTA 1 pass start, consumer warp 0 done, block-reduced, producer done, last consumer
   warp done, last warp at the block reduction, then the master's grid reduction:
   started, rows loaded, warps combined, folded} (globaltimer ns);
   row 0 = kernel start, row e =
   grid epoch e (phase -1 start, 0 lambda0/init, 1 scan, 2 breakpoint, 6 snap).
   Returns rows copied. */
int cqk_get_timeline(cqk_handle *h, long long *out, int32_t max_rows);
/* Copy the last solve's per-evaluation trace rows (4 doubles each). */
int cqk_get_trace(cqk_handle *h, double *out, int32_t max_rows);

/* CQK ----------------------------------------------------------------------- */
/* validate(inst)  core.py:126-165 */
int cqk_validate_f64(cqk_handle *h, int mem, const double *d, const double *a,
                     const double *b, const double *l, const double *u, int64_t n,
                     double r, cqk_result *res);
/* initial_multiplier(inst, xbar)  core.py:237-257 ; xbar may be NULL */
int cqk_initial_multiplier_f64(cqk_handle *h, int mem, const double *d, const double *a,
                               const double *b, const double *l, const double *u,
                               int64_t n, double r, const double *xbar, double *lam0);
/* _phi_scan / eval_phi(inst, lam, idx)  core.py:182-225.  idx may be NULL (all
   n).  out4 = {value, dminus, dplus, abs_bx}; at_lower/at_upper (length m) may
   be NULL. */
int cqk_phi_f64(cqk_handle *h, int mem, const double *d, const double *a,
                const double *b, const double *l, const double *u, int64_t n,
                const int64_t *idx, int64_t m, double lam, double *out4,
                uint8_t *at_lower, uint8_t *at_upper);
/* eval_x(inst, lam, idx)  core.py:168-179 -> x[m] */
int cqk_eval_x_f64(cqk_handle *h, int mem, const double *d, const double *a,
                   const double *b, const double *l, const double *u, int64_t n,
                   const int64_t *idx, int64_t m, double lam, double *x);
/* nearest_breakpoint  newton.py:129-162 ; right!=0: min bp > edge, else max bp < edge.
   *found = 0 when none exists. */
int cqk_nearest_breakpoint_f64(cqk_handle *h, int mem, const double *d, const double *a,
                               const double *b, const double *l, const double *u,
                               int64_t n, const int64_t *idx, int64_t m, double edge,
                               int right, double *bp, int32_t *found);
/* solve_cqk / jacobi_solve / par_solve_cqk  (variant in opts).  xbar may be
   NULL; x may be NULL (multiplier only). */
int cqk_solve_f64(cqk_handle *h, int mem, const double *d, const double *a,
                  const double *b, const double *l, const double *u, int64_t n,
                  double r, const cqk_options *opts, const double *xbar, double *x,
                  cqk_result *res);

/* output="sparse" (simplex.py:296-300; project_l1 simplex.py:328-331): the
   nonzero x as (index, value) pairs in increasing index order, without a
   dense x -- from the capture start's list (n >= 4e6 per rank, a support of
   at most n/64).  l1 = 1: project_l1's signed values.  idx_out / val_out hold
   cap entries (host or device memory per `mem`); *count = the number of
   nonzeros.  Returns 0, CQK_SPARSE_DENSE (the route does not apply: call the
   dense entry point), CQK_SPARSE_OVERFLOW (count > cap) or an error. */
int spx_project_sparse_f64(cqk_handle *h, int mem, const double *y, int64_t n, double r,
                           const cqk_options *opts, int l1, int64_t *idx_out, double *val_out,
                           int64_t cap, int64_t *count, cqk_result *res);

/* float32 instances (core.py:55-64 keeps float32 arrays float32): the element
   math in float -- t = (b * float(lam) + a) / d, x = clip(t, l, u), b x
   (core.py:195-200) -- with fp64 accumulation of the sums, on the
   warp-segment kernel; the fp32 tau eps32^(3/4) unless opts set one
   (newton.py:64-67).  Same contract as cqk_solve_f64 otherwise. */
int cqk_solve_f32(cqk_handle *h, int mem, const float *d, const float *a, const float *b,
                  const float *l, const float *u, int64_t n, double r, const cqk_options *opts,
                  const float *xbar, float *x, cqk_result *res);
/* float32 simplex / l1: v = y + float(lam) in float (simplex.py:207-215), x =
   max(0, y + float(lam)) in float (simplex.py:303, 333); the formula / tight
   starts (simplex_start 2 = alg2 runs as tight). */
int spx_project_f32(cqk_handle *h, int mem, const float *y, int64_t n, double r,
                    const cqk_options *opts, float *x, cqk_result *res);
int l1_project_f32(cqk_handle *h, int mem, const float *y, int64_t n, double r,
                   const cqk_options *opts, float *x, cqk_result *res);

/* Simplex / l1 ---------------------------------------------------------------- */
/* newton_project_simplex(y, r, opts, lambda0)  simplex.py:218-308.  The device
   initializer is lambda0 = min((r - sum y)/n, r - max y) (opts->simplex_start
   = 1) or the plain formula (0), clamped to >= min(-y) -- the reference's
   `lambda0=` route, simplex.py:246-250 -- unless opts->lambda0 is given.
   x may be NULL. */
int spx_project_f64(cqk_handle *h, int mem, const double *y, int64_t n, double r,
                    const cqk_options *opts, double *x, cqk_result *res);
/* project_l1(y, r)  simplex.py:311-333 (dense).  res->iterations = -1 when y is
   already inside the ball (x = copy of y). */
int l1_project_f64(cqk_handle *h, int mem, const double *y, int64_t n, double r,
                   const cqk_options *opts, double *x, cqk_result *res);
/* Warm-started projections: newton_project_simplex(y, r, xbar=, sharpened=)
   (simplex.py:218-308 with the xbar-support initializer, simplex.py:65-109)
   and project_l1(y, r, xbar=) (simplex.py:311-333, sharpened, xbar = |xbar|).
   Algorithm 2 runs per chunk on the device from xbar's support (par_simplex_init
   merge, parallel.py:330-368), Algorithm 4 on its free set.  xbar: n values or
   NULL; sharpened: 0 / 1 (simplex only). */
int spx_project_warm_f64(cqk_handle *h, int mem, const double *y, int64_t n, double r,
                         const cqk_options *opts, const double *xbar, int sharpened, double *x,
                         cqk_result *res);
int l1_project_warm_f64(cqk_handle *h, int mem, const double *y, int64_t n, double r,
                        const cqk_options *opts, const double *xbar, double *x, cqk_result *res);
/* simplex_init_lambda (simplex.py:114-154; workers = 1) and par_simplex_init
   (parallel.py:330-368; workers = W chunks as _chunk_ranges): Algorithm 2 per
   chunk on the device (one thread per chunk, bit-exact recurrence) merged in
   _tree_sum order.  idx (length p) selects candidates (NULL = all n); xbar and
   sharpened as the reference.  Outputs: lambda0, |free|, free indices
   (concatenated J; may be NULL), fixed_mask (length n; may be NULL), sum over
   the free set, total jplus (for the xbar fallback; may be NULL). */
int spx_init_alg2_f64(cqk_handle *h, int mem, const double *y, int64_t n, double r,
                      const int64_t *idx, int64_t p, int64_t workers, const double *xbar,
                      int sharpened, double *lam0, int64_t *nfree, int64_t *free_idx,
                      uint8_t *fixed_mask, double *sum_free, int64_t *jplus);
/* Row-wise newton_project_simplex(Y[i], r) for `rows` independent rows of
   length `cols` (row-major).  lam/iters per row may be NULL. */
int spx_project_batched_f64(cqk_handle *h, int mem, const double *Y, int64_t rows,
                            int64_t cols, double r, const cqk_options *opts, double *X,
                            double *lam, int32_t *iters, cqk_result *res);

/* Batched rows split across GPUs (replicas, no communication):
   host Y / X (row-major), rows cut into nh contiguous blocks (block q = rows
   [rows*q/nh, rows*(q+1)/nh)), block q solved by handle hs[q] -- one host
   thread per handle, all devices concurrently.  Per-row results are those of
   spx_project_batched_f64 on the same row.  res: summed byte counters,
   device_ms = the slowest block. */
int spx_project_batched_multi_f64(cqk_handle *const *hs, int nh, const double *Y, int64_t rows,
                                  int64_t cols, double r, const cqk_options *opts, double *X,
                                  double *lam, int32_t *iters, cqk_result *res);

/* Multi-GPU (one process / handle per GPU, n sharded contiguously) -------------
   Replaces the reference's chunked fork-join (parallel.py:174-327, chunks =
   _chunk_ranges parallel.py:82-85, fixed-order _tree_sum parallel.py:62-72)
   with one rank per GPU: every Newton epoch the persistent kernel of each rank
   stores its partial-sum vector into every peer's mailbox over NVLink and
   reduces the W vectors in rank order (identical decisions on all ranks). */
/* Size of the opaque IPC handle written by cqk_comm_create (bytes). */
int cqk_comm_ipc_handle_size(void);
/* Allocate this rank's mailbox; writes its CUDA IPC handle to ipc_handle_out
   (cqk_comm_ipc_handle_size() bytes) for exchange between the processes. */
int cqk_comm_create(cqk_handle *h, int rank, int world, void *ipc_handle_out);
/* Map all ranks' mailboxes from the concatenated handles (world x size bytes). */
int cqk_comm_connect(cqk_handle *h, const void *handles);
/* Same-process ranks (e.g. several handles on one device): direct pointers. */
int cqk_comm_connect_local(cqk_handle *h, cqk_handle *const *ranks, int world);
/* Pre-allocate compaction scratch for solves of up to n elements, so that a
   later solve performs no allocation (which could synchronise the device
   while another rank's persistent kernel is running). */
int cqk_reserve(cqk_handle *h, int64_t n);
/* Cap the persistent grid (CTAs); 0 = the full device.  Lets several ranks
   share one GPU (virtual ranks) or leave SMs for other work. */
/* CQK solve engine: 0 auto (TMA pipeline from CQK_TMA_MIN_N elements per rank,
   default 65536), 1 TMA pipeline, 2 warp-segment kernel.  Results agree to
   rounding (summation order differs). */
/* Pre-allocate the host-mode staging of an n-element shard (collective solves
   with CQK_MEM_HOST must not allocate while peers wait inside the kernel). */
int cqk_reserve_host(cqk_handle *h, int64_t n);
int cqk_set_engine(cqk_handle *h, int mode);
/* Fused start of the TMA CQK solve (no explicit lambda0, no xbar): a sample
   pass estimates lambda0, then ONE pass computes lambda0 (core.py:237-257) and
   validate() and classifies every element against [est(1 - w), est(1 + w)];
   the first phi scan then reads only the elements it could not classify.
   Used from min_n elements per rank (default 4e6, CQK_FUSED_MIN_N); w =
   half_width (default 2e-3).  Results agree with the unfused solve to
   rounding (lambda0's terms share the division's reciprocal). */
int cqk_set_fused(cqk_handle *h, int64_t min_n, double half_width);
/* Direction guess of the fused start (fixing solves, default 1 = auto,
   CQK_FUSED_GUESS; from 8e6 elements per rank): the sample tiles carry all
   five arrays and stay in shared memory; once the estimate is known each CTA
   evaluates phi there over its own sample and, when its estimate of
   phi(lambda0) - r is decisive, guesses which bound the first Newton
   iteration fixes (newton.py:165-206).  The fused pass then also writes that
   CTA's elements the fixing would not drop; when the side scan confirms the
   direction, the CTAs that guessed it adopt those survivors as their working
   set (the first full re-read is avoided).  0 off, 2 / 3 force +1 / -1 in
   every CTA (tests: a wrong guess is simply not adopted).  Results agree with
   mode 0 to rounding (summation order differs). */
int cqk_set_fused_guess(cqk_handle *h, int mode);
/* A/B switches of the persistent kernels (defaults 0 = the measured best;
   the environment variables of the same names set them at cqk_create):
   bit 0 CQK_MASTER_STEP (master + release grid step instead of masterless),
   bit 1 CQK_STATIC_FINAL (static final-pass tiles), bit 2 CQK_TAIL=0 (no
   single-CTA simplex tail), bit 3 CQK_SPX_CAPTURE=0 (no simplex / l1 capture
   start: pass 0 and a full first scan), bit 4 (tests) a capture threshold
   that always fails its check (the fallback to a full first scan).  Results
   are bit-identical for bits 0-2 and agree to rounding for bits 3-4. */
int cqk_set_switches(cqk_handle *h, int flags);
int cqk_set_grid_limit(cqk_handle *h, int max_ctas);
/* Sharded solve_cqk / jacobi_solve / par_solve_cqk: this rank's shard
   [offset, offset + n_local) of an n_total-element instance.  All ranks call
   it collectively with identical r and options; x (length n_local) receives
   this rank's part of the solution; res is identical on every rank except the
   byte counters, which are per rank. */
int cqk_solve_sharded_f64(cqk_handle *h, int mem, const double *d, const double *a,
                          const double *b, const double *l, const double *u, int64_t n_local,
                          int64_t offset, int64_t n_total, double r, const cqk_options *opts,
                          const double *xbar, double *x, cqk_result *res);
/* Sharded newton_project_simplex / project_l1 (formula start over n_total). */
int spx_project_sharded_f64(cqk_handle *h, int mem, const double *y, int64_t n_local,
                            int64_t n_total, double r, const cqk_options *opts, double *x,
                            cqk_result *res);
int l1_project_sharded_f64(cqk_handle *h, int mem, const double *y, int64_t n_local,
                           int64_t n_total, double r, const cqk_options *opts, double *x,
                           cqk_result *res);

/* Device groups: one process, several GPUs ------------------------------------
   The GPU analogue of the reference's worker pool (workers= / CQK_WORKERS,
   parallel.py:52-59): a group holds one handle and rank per listed device
   (mailboxes connected, peer access enabled; a device listed k times hosts k
   ranks on 1/k of its SMs), and its solves take HOST arrays, cut n into
   contiguous shards (_chunk_ranges, parallel.py:82-85) and run every rank's
   sharded solve concurrently, one host thread per rank (each rank stages its
   own shard over its own PCIe link).  The outcome is that of the sharded
   entry points; counters are summed over ranks, device_ms is the slowest
   rank.  Python: CQK_DEVICES="0,1,..." routes host-array solve_cqk /
   jacobi_solve / par_solve_cqk / newton_project_simplex / project_l1 calls
   here. */
typedef struct cqk_group cqk_group;
int cqk_group_create(cqk_group **out, const int *devices, int ndev);
int cqk_group_destroy(cqk_group *g);
int cqk_group_size(const cqk_group *g);
int cqk_solve_group_f64(cqk_group *g, const double *d, const double *a, const double *b,
                        const double *l, const double *u, int64_t n, double r,
                        const cqk_options *opts, const double *xbar, double *x, cqk_result *res);
int spx_project_group_f64(cqk_group *g, const double *y, int64_t n, double r,
                          const cqk_options *opts, double *x, cqk_result *res);
int l1_project_group_f64(cqk_group *g, const double *y, int64_t n, double r,
                         const cqk_options *opts, double *x, cqk_result *res);

/* On-device instances --------------------------------------
   gen_cqk(family, n, seed) (instances.py:43-70) straight into device arrays,
   bit-identical to the reference's stream (GF(2) jump per thread); r from
   device sums of b.l and b.u.  family: 0 uncorrelated, 1 weakly, 2 correlated. */
int cqk_gen_cqk_device(cqk_handle *h, int family, int64_t n, uint64_t seed, double *d,
                       double *a, double *b, double *l, double *u, double *r);
/* Elements [lo, hi) of the same instance (a rank's shard), with the shard's
   b.l and b.u sums; combine the shards' sums (rank order) with
   cqk_gen_cqk_r of include/cqk_instances.h. */
int cqk_gen_cqk_device_range(cqk_handle *h, int family, int64_t n, uint64_t seed, int64_t lo,
                             int64_t hi, double *d, double *a, double *b, double *l, double *u,
                             double *bl, double *bu);
/* gen_simplex_y("simplex-u01", n, seed) (instances.py:73-86) into device y. */
int cqk_gen_simplex_u01_device(cqk_handle *h, int64_t n, uint64_t seed, double *y);

/* Diagnostics ------------------------------------------------------------------ */
/* Read-only HBM streaming ceiling: `narr` (1..5) device arrays of n doubles
   streamed by a bulk-copy pipeline (one CTA per SM) `reps` times after one
   warm-up; best GB/s (and ms).  The roofline's second denominator (SURVEY
   8(d): the phi passes are reads, MEASURED_PEAKS.json's peak is a copy).
   `arrays` is a host array of device pointers. */
int cqk_read_peak_f64(cqk_handle *h, const double *const *arrays, int narr, int64_t n, int reps,
                      double *gbs_best, double *ms_best);
/* Bitwise check of the solver's shared-reciprocal division against the IEEE
   library division on `count` random operand pairs (mode 0: exponents in
   [-500, 500]; 1: solver-like ranges; 2: quotients at rounding boundaries). */
int cqk_selftest_division(cqk_handle *h, uint64_t seed, int64_t count, int mode,
                          uint64_t *mismatches, double *example2);

#ifdef __cplusplus
}
#endif
#endif
