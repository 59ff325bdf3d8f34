/*
 * fabm.h — C ABI of the B200-native fractional Adams–Bashforth–Moulton (ABM)
 * history engine (libfabm.so).
 *
 * The reference package `fodeabm` has no FFI: its drop-in boundary is the
 * Python solver call
 *
 *     solve_serial(problem: FractionalProblem, grid: GridSpec) -> Trajectory
 *         (/root/reference/pkg/src/fodeabm/serial.py:114-176)
 *
 * plus the strategy dispatch strings (bench.py:43-51, cli.py:86-94) and the
 * weight seam `precompute_weights` (core.py:134-154, serial.py:130).  Every
 * entry point below replaces one of those; the replaced interface is cited
 * next to each declaration.  Signatures use plain C types only (no torch,
 * no CUDA types): pointers are HOST pointers unless the name says `_device`.
 *
 * Conventions carried over from the reference:
 *   - errors: a bad configuration returns FABM_ERR_CONFIG (the reference's
 *     ValueError, core.py:62-66,203-220; serial.py:125-129); a non-finite
 *     rhs output returns FABM_ERR_NONFINITE with the loop index `step` and
 *     t = (step+1)*h of the first failing evaluation (SolverStepError,
 *     core.py:34-43, serial.py:157-174); a stuck solve returns
 *     FABM_ERR_TIMEOUT (StrategyTimeoutError, core.py:46-47).
 *   - calls are synchronous: they return when the whole trajectory is done
 *     (SPEC.md:128); outputs are fresh caller-owned buffers.
 *   - determinism: identical inputs give bitwise identical outputs
 *     (bench.py:80-87 enforces this for every strategy).
 */
#ifndef FABM_H
#define FABM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FABM_MAX_DIM 4      /* state dimension supported by the device engine */
#define FABM_MAX_PARAMS 16  /* rhs parameters per problem */

/* status codes */
enum {
  FABM_OK = 0,
  FABM_ERR_NONFINITE = 1, /* SolverStepError: rhs returned a non-finite value */
  FABM_ERR_CONFIG = 2,    /* ValueError: bad alpha/dim/y0/grid/system */
  FABM_ERR_TIMEOUT = 3,   /* StrategyTimeoutError: device watchdog expired */
  FABM_ERR_CUDA = 4,      /* CUDA runtime failure (message in status) */
  FABM_ERR_NODEVICE = 5,  /* no usable sm_100 device */
  FABM_ERR_IO = 6         /* OSError: the output file could not be written */
};

/* which rhs evaluation failed (fabm_status.kind) */
enum {
  FABM_KIND_NONE = 0,
  FABM_KIND_INITIAL = 1,   /* f(0, y0)          core.py:226-236            */
  FABM_KIND_PREDICTOR = 2, /* f(t_{n+1}, yP)    serial.py:156-158          */
  FABM_KIND_CORRECTOR = 3  /* f(t_{n+1}, y_{n+1}) serial.py:166-168        */
};

/* device right-hand sides (systems.py:26-123 + the BASELINE.json systems) */
enum {
  FABM_SYS_CONSTANT = 0,       /* params[0..d-1] = value            systems.py:26-36  */
  FABM_SYS_POWER_LAW = 1,      /* params = {coef, expo}             systems.py:39-61  */
  FABM_SYS_LINEAR = 2,         /* params = {lam}                    systems.py:64-73  */
  FABM_SYS_HINDMARSH_ROSE = 3, /* params = {a,b,c,d,r,s,x_rest,i}   systems.py:101-123 */
  FABM_SYS_LORENZ = 4,         /* params = {sigma, rho, beta}                         */
  FABM_SYS_CHEN = 5,           /* params = {a, b, c}                                  */
  FABM_SYS_ROSSLER = 6,        /* params = {a, b, c}                                  */
  FABM_SYS_FINANCIAL = 7       /* params = {a, b, c}                                  */
};

/* weight generation modes (fabm_weights / fabm_plan_set_weights) */
enum {
  FABM_WEIGHTS_ACCURATE = 0, /* device, cancellation-free series (few ulp)          */
  FABM_WEIGHTS_FORMULA = 1,  /* device, the reference's pow formula (core.py:149-151) */
  FABM_WEIGHTS_HOST = 2      /* caller-provided table (the precompute_weights seam) */
};

/* FractionalProblem (core.py:188-236) with a device rhs tag instead of a
 * Python callable. */
typedef struct fabm_problem {
  double alpha;                     /* (0, 1]                                  */
  int32_t dim;                      /* 1..FABM_MAX_DIM                         */
  int32_t system;                   /* FABM_SYS_*                              */
  double params[FABM_MAX_PARAMS];
  double y0[FABM_MAX_DIM];
} fabm_problem;

/* GridSpec (core.py:157-185) plus the per-solve scalars serial.py:135-136
 * computes in Python.  The caller passes them so the device uses the very
 * same bits (CPython's math.gamma is not libm's tgamma).  A zero field is
 * filled by the library from libm. */
typedef struct fabm_grid {
  int64_t n_steps;   /* N >= 1                                       */
  double h;          /* step size                                    */
  double h_alpha;    /* h ** alpha                  (serial.py:135)  */
  double inv_gamma2; /* 1 / Gamma(alpha + 2)        (serial.py:136)  */
  double gamma1;     /* Gamma(alpha + 1)            (core.py:146)    */
  double gamma2;     /* Gamma(alpha + 2)            (core.py:147)    */
} fabm_grid;

typedef struct fabm_status {
  int32_t code;      /* FABM_OK / FABM_ERR_*                         */
  int32_t kind;      /* FABM_KIND_* for FABM_ERR_NONFINITE           */
  int64_t step;      /* loop index n of the failing step             */
  double t;          /* (n + 1) * h                                  */
  int64_t index;     /* batch: lowest failing trajectory (else -1)   */
  char message[240];
} fabm_status;

typedef struct fabm_stats {
  double kernel_ms;        /* engine kernel, CUDA events on the engine stream   */
  double weights_ms;       /* weight-generation kernel                          */
  int64_t steps;           /* steps taken                                       */
  int64_t history_fma;     /* algorithmic history FMAs per trajectory = d*N^2   */
  int64_t bulk_tiles;      /* Toeplitz tiles processed by the bulk agents       */
  int64_t leader_wait_ns;  /* time the stepper spent waiting on handoffs        */
  int64_t leader_throttle_ns; /* time the stepper waited for ring consumers     */
  int32_t bulk_ctas;       /* CTAs running bulk agents                          */
  int32_t block;           /* history block B                                   */
  int32_t window_blocks;   /* stepper window L (blocks)                         */
  int32_t segment;         /* source blocks per bulk unit (fixed by n_steps)    */
  int64_t bulk_claims;     /* bulk units computed by an agent other than the owner */
} fabm_stats;

typedef struct fabm_plan fabm_plan;

/* ---- library ---------------------------------------------------------- */
const char* fabm_version(void);
int fabm_device_count(void);

/* ---- weights: replaces precompute_weights (core.py:134-154) -----------
 * Fills b, a, c (host buffers of n_steps+1 doubles) using the device
 * generator in `mode` (FABM_WEIGHTS_ACCURATE or FABM_WEIGHTS_FORMULA). */
int fabm_weights(double alpha, int64_t n_steps, int mode, double gamma1,
                 double gamma2, double* b, double* a, double* c,
                 fabm_status* status);

/* ---- one trajectory: replaces solve_serial (serial.py:114-176) ---------
 * states and f_cache are host buffers of (n_steps+1)*dim doubles, row n =
 * y_n / f(t_n, y_n) (Trajectory, serial.py:36-64).  When weight_mode is
 * FABM_WEIGHTS_HOST, b/a/c point at n_steps+1 doubles each (the table the
 * reference's precompute_weights returned); otherwise they may be NULL. */
int fabm_solve(const fabm_problem* problem, const fabm_grid* grid,
               int weight_mode, const double* b, const double* a,
               const double* c, double* states, double* f_cache,
               fabm_status* status);

/* ---- plan API: device-resident buffers, for repeated solves/benchmarks - */
fabm_plan* fabm_plan_create(const fabm_problem* problem, const fabm_grid* grid,
                            int device, fabm_status* status);
int fabm_plan_set_weights(fabm_plan* plan, int weight_mode, const double* b,
                          const double* a, const double* c, fabm_status* status);
/* upload y0 (host) for this run; NULL keeps the plan's current y0 */
int fabm_plan_set_y0(fabm_plan* plan, const double* y0, fabm_status* status);
/* run the engine on the plan's stream; inputs must already be resident */
int fabm_plan_run(fabm_plan* plan, double timeout_s, fabm_status* status);
int fabm_plan_download(fabm_plan* plan, double* states, double* f_cache,
                       fabm_status* status);
/* final state y_N only (d doubles) — the small D2H read of the bench */
int fabm_plan_download_last(fabm_plan* plan, double* y_last, fabm_status* status);
int fabm_plan_stats(const fabm_plan* plan, fabm_stats* stats);
void fabm_plan_destroy(fabm_plan* plan);

/* Stream the next runs' trajectory (states, f_cache: (n_steps+1)*dim doubles
 * each) straight into pinned host memory while the kernel runs, so no D2H
 * copy follows the solve (how solve_gpu returns the Trajectory of
 * serial.py:36-64 as fresh host arrays; no reference counterpart).  The buffers must be mapped pinned memory, e.g.
 * from fabm_host_alloc, and stay valid until the plan is reset with NULLs or
 * destroyed.  Both NULL: back to device-only output (fabm_plan_download). */
int fabm_plan_set_host_output(fabm_plan* plan, double* states, double* f_cache,
                              fabm_status* status);
void* fabm_host_alloc(int64_t bytes);   /* mapped, portable pinned memory; NULL on failure */
void fabm_host_free(void* ptr);

/* Cap the bulk-agent CTAs of the next runs (n_ctas <= 0: the default, one
 * CTA per SM besides the stepper).  Results do not depend on it (the unit
 * partition and the reduction order depend on n_steps only); the parity
 * tests use it to put many target blocks on each agent at small n_steps.
 * No reference counterpart (the reference's worker count, parallel/block.py:
 * 44-51, sets its partition instead). */
int fabm_plan_set_bulk_ctas(fabm_plan* plan, int n_ctas, fabm_status* status);

/* Zero the run flags of a plan.  fabm_plan_run does this itself, except on a
 * plan attached to peer shards: there every rank calls fabm_plan_reset, then
 * the ranks barrier, then every rank calls fabm_plan_run. */
int fabm_plan_reset(fabm_plan* plan, fabm_status* status);

/* ---- one trajectory sharded over the GPUs of a node (BASELINE config 5) ---
 * Replaces the reference's block-partitioned ParallelABM (parallel/block.py:
 * 44-236 with partition.py:54-74): instead of per-step partial sums from lower
 * workers, every GPU hosts bulk agents that compute bulk units (fixed source
 * segments of a target block), so the exchange is one NVLink store of each
 * unit's partial sum into rank 0's slots -- reduced there once per target
 * block in a fixed order -- plus the f history rows fanned out by rank 0's
 * stepper.  Results are bitwise equal to the single-GPU run.  One process per GPU: each rank creates a plan
 * for the same problem/grid on its own device, exports its IPC handle, the
 * ranks all-gather the handles (rank order), and each calls attach. */
#define FABM_IPC_HANDLE_BYTES 64
#define FABM_MAX_SHARDS 8
int fabm_plan_ipc_handle(fabm_plan* plan, void* handle_out, fabm_status* status);
int fabm_plan_attach_shards(fabm_plan* plan, int n_shards, int rank, const void* handles,
                            fabm_status* status);
/* Close the peer mappings (every rank, then barrier, then destroy: an arena
 * must outlive the peers' mappings of it). */
int fabm_plan_detach_shards(fabm_plan* plan, fabm_status* status);
/* On rank 0 of an attached plan: run every shard's agents in THIS launch
 * (as fabm_plan_set_virtual_shards does), with the peers' arenas -- their f
 * copies and control blocks -- used through their CUDA IPC mappings.  Only
 * rank 0 launches, so no kernels on different launches wait on each other:
 * the cross-process IPC path (handle export, open, system-scope flags and
 * stores into a peer's memory, detach) runs where only one GPU is available
 * (tests/test_gpu_sharded_ipc.py).  on = 0 restores the per-rank launches. */
int fabm_plan_emulate_shards(fabm_plan* plan, int on, fabm_status* status);
/* This plan's own control block after a run: source blocks released into it
 * (src_done) and Toeplitz tiles its shard's agents processed. */
int fabm_plan_shard_counters(const fabm_plan* plan, int64_t* src_done, int64_t* bulk_tiles,
                             fabm_status* status);
/* One-GPU emulation of an n-shard run: separate per-shard f copies, control
 * blocks and scratch on this device, agent CTA b serving shard (b-1) % n.
 * Exercises the sharded protocol where only one GPU is available. */
int fabm_plan_set_virtual_shards(fabm_plan* plan, int n_shards, fabm_status* status);

/* ---- batch: many independent trajectories (BASELINE config 4) ----------
 * A sweep of `count` problems is `count` solve_serial calls in the reference
 * (serial.py:114-176).  problems[count] and grids[count] must share dim,
 * system, n_steps and h; alpha, y0, params and the per-solve scalars may
 * differ.  Weights are generated on the device per trajectory (ACCURATE).
 * Outputs (host, trajectory-major, any may be NULL):
 *   states, f_cache : count*(n_steps+1)*dim doubles
 *   y_last          : count*dim doubles (y_N of every trajectory)
 * A non-finite rhs stops that trajectory only; the status reports the
 * lowest failing index (status.index), its step and t. */
int fabm_solve_batch(const fabm_problem* problems, const fabm_grid* grids,
                     int64_t count, int device, double* states,
                     double* f_cache, double* y_last, double* kernel_ms,
                     fabm_status* status);

/* ---- trajectory CSV output: replaces write_trajectory_csv (cli.py:97-105) --
 * Bytes identical to the reference's Python loop: header "t,y0,..,y{d-1}\n",
 * then one row per time point, every value as CPython's f"{v:.17g}"
 * (correctly rounded, ties to even, trailing zeros removed).  The values are
 * formatted on the GPU (csrc/csv_format.cuh).
 *   states : host, n_rows * dim doubles (Trajectory.states, row-major)
 *   t      : host, n_rows doubles (Trajectory.t), or NULL for t[n] = n * h
 *            (GridSpec.times(), core.py:179-181)
 *   kernel_ms (optional out): device time of the formatting kernels
 * fabm_format_csv writes into a caller buffer: if out_cap is too small it
 * returns FABM_ERR_CONFIG with *n_bytes = the size needed (out may be NULL).
 * fabm_write_csv creates/truncates `path` like open(path, "w") and returns
 * FABM_ERR_IO if it cannot be written. */
int fabm_format_csv(const double* states, const double* t, int64_t n_rows,
                    int32_t dim, double h, int device, char* out,
                    int64_t out_cap, int64_t* n_bytes, double* kernel_ms,
                    fabm_status* status);
int fabm_write_csv(const char* path, const double* states, const double* t,
                   int64_t n_rows, int32_t dim, double h, int device,
                   int64_t* n_bytes, double* kernel_ms, fabm_status* status);
/* the CSV of the plan's last run straight from its device-resident states
 * (no D2H of the trajectory; t[n] = n * h) */
int fabm_plan_write_csv(fabm_plan* plan, const char* path, int64_t* n_bytes,
                        double* kernel_ms, fabm_status* status);

/* ---- analytic oracle on the device: replaces mittag_leffler (verify.py:28-64)
 * E_alpha(z) for n pairs (host arrays alpha[n], z[n] -> out[n]), the
 * reference's log-space power series with Kahan summation, one thread per
 * pair.  codes[n] (optional): 0 ok; 1 invalid argument (the reference's
 * ValueError: alpha outside (0, 1], |z| > 10 or z not finite; out = nan);
 * 2 a term overflowed (out = +-inf, as the reference returns); 3 no
 * convergence in 20000 terms (the reference's ArithmeticError). */
int fabm_mittag_leffler(const double* alpha, const double* z, int64_t n,
                        int device, double* out, int32_t* codes,
                        fabm_status* status);

/* ---- single-step ops: replace step_predictor / step_corrector ------------
 * (serial.py:74-111).  For each requested step index ns[i] (0 <= n <
 * grid.n_steps), from the prefix f_cache[0..n] (host, n_rows x dim):
 *   yp_out[i] = y0 + h^a * sum_{k<=n} b_{n-k} f_k                 (predictor)
 *   y_out[i]  = y0 + h^a * ((c_n f_0 + sum_{1<=k<=n} a_{n-k} f_k)
 *                           + f(t_{n+1}, y_pred[i]) / Gamma(a+2)) (corrector)
 * y_pred NULL uses the computed predictor (one full PECE step).  b/a/c hold
 * n_weights entries (a WeightTable).  err_out[i]: 0 ok; 1 the predicted state
 * is non-finite; 2 the rhs returned a non-finite value (both are the
 * reference's SolverStepError(step=n, t=(n+1)h); y_out is nan there).  An
 * index out of range is FABM_ERR_CONFIG (the reference's ValueError). */
int fabm_step_pc(const fabm_problem* problem, const fabm_grid* grid,
                 const double* b, const double* a, const double* c,
                 int64_t n_weights, const double* f_cache, int64_t n_rows,
                 const int64_t* ns, int64_t count, const double* y_pred,
                 double* yp_out, double* y_out, int32_t* err_out, int device,
                 fabm_status* status);

/* Return the device memory that batch solves keep cached in the device's
 * stream-ordered pool (fabm_solve_batch allocates from it so repeated sweeps
 * skip cudaMalloc/cudaFree).  Resource management only; no reference
 * counterpart. */
int fabm_trim_memory(int device);

/* ---- microbenchmarks used by bench.py for the roofline denominator ----- */
/* measured FP64 FMA throughput (FMA/s) of a DFMA-bound loop on `device` */
double fabm_measure_dfma_peak(int device);

#ifdef __cplusplus
}
#endif
#endif /* FABM_H */
