/*
 * pt_b200.h -- C ABI of the B200-native online polarized-traces solve.
 *
 * This is the drop-in boundary for the reference's online GMRES stage
 * (helmsweep, arXiv 1410.5910).  Every entry point below replaces one
 * reference interface; the citation is file:line in the reference package
 * (pkg/src/helmsweep/).  Plain C types only: complex numbers are
 * interleaved (re, im) doubles, layout-identical to numpy complex128 and
 * cuDoubleComplex.  Vectors passed to the apply/solve calls are DEVICE
 * pointers (cudaMalloc'd, or torch CUDA tensors' data_ptr()); the upload
 * arrays of pt_create and the *_host calls take HOST pointers.
 *
 * All functions return 0 on success, PT_EINVAL (-1) for a shape/layout
 * error (the reference raises ValueError) and PT_ECUDA (-2) for a CUDA
 * failure, PT_ENONFINITE (-3) when GMRES meets non-finite values (the
 * reference raises RuntimeError, solver.py:255-258); pt_last_error()
 * returns the message of the last failure on the calling thread.
 *
 * Calls are stream-ordered on the given stream (NULL = legacy default).
 * The programs of one handle share its dependency counters and scratch
 * vectors, so a call on a different stream than the handle's previous call
 * first waits for that call (an event); a handle must not be used from two
 * threads at once.
 */
#ifndef PT_B200_H
#define PT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PT_ABI_VERSION 1

#define PT_OK 0
#define PT_EINVAL (-1)
#define PT_ECUDA (-2)
#define PT_ENONFINITE (-3)

typedef void *pt_stream; /* a cudaStream_t */
typedef struct pt_handle pt_handle;
typedef struct pt_gmres_ws pt_gmres_ws;

/* Kernel storage formats of BlockEntry.kernel (trace_system.py:145-150). */
#define PT_KERNEL_DENSE 0 /* ndarray: m x m row-major complex128        */
#define PT_KERNEL_PLR 1   /* PLRSparseForm: quadtree leaves (plr.py:239) */

/* Shape of the polarized ("jump") interface system
 * (trace_system.py:368-472): n_block_rows = 2*nt block rows and columns of
 * m x m blocks, nt = 2L-2 trace blocks per half. */
typedef struct {
  int64_t m;            /* interface width nx + 2*n_pml                  */
  int64_t n_block_rows; /* 2*nt; must be even                            */
  int32_t kernel_format;/* PT_KERNEL_DENSE or PT_KERNEL_PLR              */
  int32_t n_kernels;    /* distinct kernel objects shared by the entries */
} pt_layout;

/* One BlockEntry: y[row] += scale * K[kernel] @ x[col] + eye * x[col]
 * (trace_system.py:159-168); kernel = -1 is a pure identity entry. */
typedef struct {
  int64_t row, col, kernel;
  double scale_re, scale_im;
  double eye_re, eye_im;
} pt_entry;

/* One PLR leaf (plr.py:58-75) of kernel `kernel`, at block offset
 * (row_off, col_off) of size rows x cols and rank `rank`.  Its factors live
 * in the factor array: U*Sigma is rows x rank row-major at u_off, Vt is
 * rank x cols row-major at vt_off (offsets in complex elements).  Leaves
 * of one kernel must tile its m x m block; rank-0 leaves may be omitted. */
typedef struct {
  int64_t kernel, row_off, col_off, rows, cols, rank, u_off, vt_off;
} pt_leaf;

/* GmresConfig (solver.py:71-80) + PreconditionerConfig.n_it (:59-68). */
typedef struct {
  double rel_tol;   /* converged when rel residual <= rel_tol           */
  int32_t max_iter; /* no restart (solver.py:231)                        */
  int32_t n_it;     /* Gauss-Seidel sweeps per preconditioner apply      */
} pt_gmres_config;

/* Flags of SolveReport.flag (solver.py:96-107, :265-289). */
#define PT_FLAG_CONVERGED 0
#define PT_FLAG_BREAKDOWN 1
#define PT_FLAG_STAGNATION 2
#define PT_FLAG_MAXITER 3

/* SolveReport subset filled by the device solve.  residual_history must
 * point to max_iter doubles (host memory) or be NULL. */
typedef struct {
  int32_t iterations;
  int32_t flag;
  int32_t converged;
  int32_t nonfinite; /* 1 if GMRES stopped on a non-finite apply */
  double true_residual;
  double beta;       /* ||M^-1 b|| */
  double *residual_history;
} pt_report;

/* ---- operator handle ----------------------------------------------------
 * Upload the offline operator once (replaces OfflineState.pol/perm/d/r,
 * solver.py:110-129, built by assemble_polarized + split_DR,
 * trace_system.py:368-524).  dense: n_kernels*m*m complex (host) or NULL;
 * leaves/factors: PLR tables (host) or NULL.  perm is sweep_permutation
 * (trace_system.py:353-365) in natural block-row indices.
 * device = PT_DEVICE_HOST builds the host-side tables only (B200 launch
 * shape assumed, dense may be NULL): such a handle answers pt_plan_stats and
 * pt_exec_info, everything else returns PT_EINVAL. */
#define PT_DEVICE_HOST (-1) /* pt_create device: plan-only handle, no GPU */
int pt_create(const pt_layout *layout, const pt_entry *entries,
              int64_t n_entries, const int64_t *perm, const double *dense,
              const pt_leaf *leaves, int64_t n_leaves, const double *factors,
              int64_t n_factor_complex, int device, pt_handle **out);
int pt_destroy(pt_handle *h);

/* y = pol @ x   (BlockInterfaceMatrix.matvec, trace_system.py:219-226). */
int pt_apply_A(pt_handle *h, const double *x, double *y, pt_stream stream);

/* z = preconditioner_apply(n_it sweeps from zero)  (solver.py:223-228). */
int pt_apply_M(pt_handle *h, const double *r, double *z, int32_t n_it,
               pt_stream stream);

/* w = M^-1 (A x): one GMRES iteration's preconditioned matvec
 * (solver.py:254) as ONE fused launch -- the sweeps start on A's output
 * blocks as they are produced. */
int pt_apply_AM(pt_handle *h, const double *x, double *w, int32_t n_it,
                pt_stream stream);

/* u_out = D^-1 (P rhs - R u_in)   (gs_sweep, solver.py:203-220). */
int pt_gs_sweep(pt_handle *h, const double *rhs, const double *u_in,
                double *u_out, pt_stream stream);

/* Left-preconditioned GMRES on the device: x = solution, report filled
 * (gmres_solve, solver.py:231-295, with CGS2 + Givens in place of MGS +
 * lstsq).  b, x device pointers.  Synchronises the stream once. */
int pt_gmres(pt_handle *h, const double *b, double *x,
             const pt_gmres_config *cfg, pt_report *report, pt_stream stream);

/* Same with HOST b/x: the H2D copy, the solve and the D2H copy all happen
 * inside (the gmres stage of solve_helmholtz, solver.py:376-397). */
int pt_gmres_host(pt_handle *h, const double *b_host, double *x_host,
                  const pt_gmres_config *cfg, pt_report *report,
                  pt_stream stream);

/* Batched independent solves of nrhs right-hand sides stored column after
 * column (b[s*N ...]); reports[s] per RHS (the per-source loop of
 * cli.py:380-409, one gmres_solve per source, solver.py:231-295).  Dense
 * operators run up to 64 sources in lockstep: each kernel row is read once
 * per iteration for all of them and every block term is a multi-RHS
 * contraction on the FP64 tensor cores; each source keeps its own status,
 * flags and iteration count.  PLR operators solve the sources one by one.
 * Returns PT_ENONFINITE (after filling every report) if any source met
 * non-finite values. */
int pt_gmres_batch(pt_handle *h, const double *b, double *x, int32_t nrhs,
                   const pt_gmres_config *cfg, pt_report *reports,
                   pt_stream stream);
/* Same with HOST b/x (copies inside). */
int pt_gmres_batch_host(pt_handle *h, const double *b_host, double *x_host,
                        int32_t nrhs, const pt_gmres_config *cfg,
                        pt_report *reports, pt_stream stream);

/* Multi-RHS applies on nrhs column-major device vectors (dense operators):
 * Y[:, s] = pol @ X[:, s] (trace_system.py:219-226) and
 * Z[:, s] = preconditioner_apply(R[:, s]) (solver.py:223-228) -- the
 * operators of pt_gmres_batch. */
int pt_apply_A_batch(pt_handle *h, const double *x, double *y, int32_t nrhs,
                     pt_stream stream);
int pt_apply_M_batch(pt_handle *h, const double *r, double *z, int32_t nrhs,
                     int32_t n_it, pt_stream stream);

/* ---- generic GMRES workspace (callable operators) ------------------------
 * The reference's gmres_solve takes arbitrary callables apply_A/apply_Minv.
 * These entry points run the device Arnoldi/Givens machinery while the
 * caller applies its own operators between steps. */
int pt_gmres_ws_create(int64_t n, int32_t max_iter, int device,
                       pt_gmres_ws **out);
int pt_gmres_ws_destroy(pt_gmres_ws *ws);
/* device pointer to basis column j (length n), for the caller's applies */
double *pt_gmres_ws_basis(pt_gmres_ws *ws, int32_t j);
/* mb = M^-1 b already computed by the caller: beta = ||mb||, V0 = mb/beta.
 * *beta_out receives beta (0 => x = 0, converged). */
int pt_gmres_ws_begin(pt_gmres_ws *ws, const double *mb, double *beta_out,
                      pt_stream stream);
/* w = M^-1 A v_j has been written to basis column j+1 by the caller:
 * CGS2 + Givens + flags.  *stop_out = 1 when the loop must end; status
 * fields land in the report (residual_history appended). */
int pt_gmres_ws_step(pt_gmres_ws *ws, int32_t j, double rel_tol,
                     int32_t max_iter, pt_report *report, int32_t *stop_out,
                     pt_stream stream);
/* x = V[:, :k] y after the loop (k = report->iterations). */
int pt_gmres_ws_finish(pt_gmres_ws *ws, int32_t k, double *x,
                       pt_stream stream);

/* ---- instrumentation -------------------------------------------------------
 * With timing enabled every executor launch (operator apply / sweep /
 * fused A->M iteration) is bracketed by CUDA events on its stream;
 * pt_exec_stats synchronises the device and returns the summed device time,
 * the launch count and the algorithmic kernel bytes of those launches
 * (SURVEY.md §8(d)), then resets the accumulators. */
int pt_exec_timing(pt_handle *h, int32_t enable);
int pt_exec_stats(pt_handle *h, double *total_ms, int64_t *launches,
                  int64_t *algo_bytes);

/* Run one operator program (kind 0 = A-apply, 1 = n_it-sweep preconditioner,
 * 2 = fused A->M iteration, 3 = one sweep with u_in = in) with a per-task
 * timeline: rec[PT_TRACE_WORDS*q ...] = {type, out slot, out offset, r0, r1,
 * terms, t_grab, t_ready (dependencies met), t_done (globaltimer ns), SM id |
 * CTA index << 16,
 * t_consumers_start, group, t_staged, pieces, t_issue[8] (producer issued
 * operator piece k), t_landed[8] (consumers saw piece k), consumer cycles
 * waiting for pieces, consumer cycles in per-piece barriers} for every task q in
 * queue order (0 = not recorded).  Profiling aid; synchronises. */
#define PT_TRACE_WORDS 32
int pt_trace_program(pt_handle *h, int32_t kind, int32_t n_it, const double *in,
                     double *out, int64_t *rec, int64_t cap, int64_t *n_out);

/* Executor launch shape: CTAs (cooperative grid), dynamic smem per CTA and
 * the complex capacity of one operator staging buffer half. */
int pt_exec_info(const pt_handle *h, int32_t *grid, int64_t *smem_bytes,
                 int64_t *half_elems);

/* Host-side plan of one program (kind as in pt_trace_program) without
 * running it: stats[0..11] = {tasks, T_PLR tasks, Y_PLR tasks, Y_DENSE tasks,
 * operator pieces, metadata items, counters, algorithmic bytes, staged
 * operator bytes, max terms of a task, max pieces of a task, max items of a
 * task}.  PT_EINVAL (pt_last_error says why) if a task exceeds what the
 * executor stages.  Needs no GPU. */
#define PT_PLAN_STATS 12
int pt_plan_stats(pt_handle *h, int32_t kind, int32_t n_it, int64_t *stats);

/* Host-side task list of one program (profiling aid): rec[PT_TASK_WORDS*q
 * ...] = {type, signal counter, nwait | on-sweep-chain << 16, pieces, r0, r1,
 * out slot | items << 8, staged operator elements, (counter, target) of the
 * first 8 waits (-1: none)} in queue order. */
#define PT_TASK_WORDS 24
int pt_plan_tasks(pt_handle *h, int32_t kind, int32_t n_it, int32_t *rec,
                  int64_t cap, int64_t *n_out);

/* ---- per-layer local solves (Newton traces, volume reconstruction) --------
 * The reference solves each layer's sparse system with SuperLU on the host
 * (LocalFactorization.solve, local_solver.py:21-60) for the Newton traces
 * (newton_trace, :138-144) and the volume (reconstruct_volume, :147-176).
 * Here the host offline stage factors every layer once (Pr (P A P^T) Pc = L U
 * with a nested-dissection P) and these calls keep L and U of all layers on
 * the device and solve every layer in one pass of two sync-free sparse
 * triangular solves.  Per layer: CSR of L and U (complex values interleaved,
 * diagonal included) and the composed gathers q_in (y[k] = b[q_in[k]], b in
 * the layer's natural (z, x) order) and q_out (x[r] = z[q_out[r]]). */
typedef struct pt_local pt_local;
typedef struct {
  int64_t dim;                 /* nze * nxe unknowns of the layer           */
  int64_t nze, nxe;            /* layer grid incl. the z pads (local_solver) */
  int64_t n_layer, n_pml;      /* interior rows, pad rows on each side      */
  const int64_t *l_ptr;        /* dim + 1 */
  const int32_t *l_col;
  const double *l_val;         /* complex */
  const int64_t *u_ptr;
  const int32_t *u_col;
  const double *u_val;
  const int64_t *q_in, *q_out; /* dim each, layer-local indices */
  /* optional: the factor order's nested-dissection blocks (leaf blocks and
   * separators, contiguous rows): block k is rows [block_ptr[k],
   * block_ptr[k+1]).  With them every block is solved in two parallel steps
   * through the inverse of its diagonal block (formed at create); without
   * (n_blocks = 0), one row at a time. */
  int64_t n_blocks;
  const int64_t *block_ptr;    /* n_blocks + 1 */
} pt_local_layer;
/* layers in depth order (layer l's interior rows follow layer l-1's) */
int pt_local_create(const pt_local_layer *layers, int32_t n_layers, int device,
                    pt_local **out);
int pt_local_destroy(pt_local *h);
/* rows = total unknowns, factor_nnz = stored entries of L and U, levels =
 * dependency depth of the triangular solves */
int pt_local_info(const pt_local *h, int64_t *rows, int64_t *factor_nnz,
                  int32_t *l_levels, int32_t *u_levels);
/* x = H^-1 b for every layer (layers concatenated, natural order; device) */
int pt_local_solve(pt_local *h, const double *b, double *x, pt_stream stream);
/* Newton traces of source f (extended grid, nz_ext x nxe, device):
 * traces[l][d][c] at local depths d = (0, 1, n, n+1) (newton_trace) and/or
 * the polarized right-hand side (polarized_rhs, trace_system.py:475-484;
 * jump = 0: the extrapolation variant's zero bottom half).  Either output
 * may be NULL (not both). */
int pt_local_newton(pt_local *h, const double *f, double *traces, double *rhs,
                    int32_t jump, pt_stream stream);
/* Volume of every layer (reconstruct_volume with the interface forcing of
 * the traces x_down + x_up of the GMRES solution x; solver.py:403-426):
 * u (nz x nxe interior rows, device). */
int pt_local_reconstruct(pt_local *h, const double *f, const double *x,
                         double h_step, double *u, pt_stream stream);
const char *pt_local_last_error(void);

/* ---- misc ----------------------------------------------------------------*/
const char *pt_last_error(void);
int32_t pt_abi_version(void);
/* number of kernels this library has launched since load (the nodes of
 * graph-resident solves are counted per execution) */
int64_t pt_launch_count(void);
/* 1 for the checked build (libpt_b200_check.so, -DPT_CHECK=1: the executor
 * asserts its index/capacity invariants and bounds every spin loop, trapping
 * with a record appended to pt_last_error()), 0 for the release build */
int32_t pt_checked_build(void);
/* algorithmic bytes of one A-apply / one n_it-sweep preconditioner apply
 * (distinct kernels read once) */
int64_t pt_bytes_apply_A(const pt_handle *h);
int64_t pt_bytes_apply_M(const pt_handle *h, int32_t n_it);

#ifdef __cplusplus
}
#endif
#endif /* PT_B200_H */
