// Multi-right-hand-side ("batched") online solve: BW independent GMRES runs
// in lockstep over one operator (the reference loops
// over sources one solve at a time, cli.py:380-409).
//
// Batched vectors hold BW right-hand sides side by side: element (i, s) of an
// N x BW block is at [i * BW + s] (complex).  Each operator kernel row is then
// read once per apply for all BW sources, and every block term becomes a
// (rows x m) . (m x BW) complex contraction on the FP64 tensor cores (DMMA,
// mma.sync m8n8k4 .f64): FP64-compute-bound instead of HBM-bound.
#pragma once
#include "pt_device.cuh"
#include "pt_gmres.cuh"

namespace pt {

constexpr int BW = 64;           // right-hand sides per batch (columns)
constexpr int BT_ROWS = 8;       // output rows of a batched task (8 or 16; PT_BATCH_ROWS; 8 measured faster at c5)
constexpr int BT_KC = 16;        // kernel columns per staged chunk
constexpr int BT_THREADS = 256;  // 8 warps: 2 row groups x 4 column groups
constexpr int BT_TERMS = 16;     // kernel terms of one task
constexpr int BT_EYES = 4;       // identity terms of one task
constexpr int BT_CTAS_PER_SM = 3;
constexpr int BRED_BLOCKS = 296;  // row ranges of the batched reductions (fixed: deterministic)

struct BExecArgs {
  const DevTask* tasks;  // queue order
  const DevTerm* terms;
  const DevEye* eyes;
  const DevWait* waits;
  int* ctr;   // producer-group counters
  int* head;  // queue head
  double2* slot[N_SLOTS];  // batched vectors (offsets of the plan scale by BW)
  const double2* dense;    // kernel pool, n_kernels x m x m row-major
  int n_tasks;
  int m;
  const int* stop;  // launch skipped when *stop != 0 (all sources stopped)
  // iteration-relative basis (GMRES loop in a graph): SLOT_IN = vbase +
  // (*iter) * vstride, SLOT_OUT = SLOT_IN + vstride
  const int* iter;
  double2* vbase;
  int64_t vstride;
};

// batched GMRES state (per-source status, rotations and history)
struct BGmresDev {
  int64_t n;      // rows N of one source
  int max_iter;
  int nrhs;       // live columns; columns >= nrhs are zero padding
  double2* V;     // (max_iter + 1) blocks of n x BW
  double2* P;     // BRED_BLOCKS x (max_iter + 1) x BW partials
  double2* h1;    // (max_iter + 1) x BW
  double2* h2;
  double2* R;     // per source: (max_iter + 1) x max_iter column-major
  double2* g;     // per source: max_iter + 1
  double* cs;     // per source: max_iter
  double2* sn;
  double* hist;   // per source: max_iter
  double2* y;     // per source: max_iter
  double* inv;    // BW: scale of the new basis column (0: stopped)
  DevStatus* st;  // BW statuses
  int* ctl;       // [0] iteration j, [1] all stopped, [2] any non-finite
};

// one batched program launch (persistent, grid = bexec_grid())
// tiles: rows x cols = 16 x 64, 8 x 64 or 16 x 32 (cols < 64: tasks carry
// their first source column in DevTask::c0)
cudaError_t bexec_launch(const BExecArgs& a, int grid, int rows, int cols, cudaStream_t s);
int bexec_grid(int device, int rows, int cols);
cudaError_t bexec_setup();

// batched GMRES steps (graph-capturable; see pt_batch.cu)
void bg_begin(const BGmresDev& g, cudaGraphConditionalHandle cond, cudaStream_t s);
void bg_step(const BGmresDev& g, double rel_tol, int max_iter, cudaGraphConditionalHandle cond,
             cudaStream_t s);
void bg_finish(const BGmresDev& g, double2* x, cudaStream_t s);
void bg_resid(const BGmresDev& g, const double2* b, const double2* ax, cudaStream_t s);
cudaError_t bg_setup(int max_iter);
// column-major sources (src[c * n + i], c < ncols) <-> batched block
void b_pack(const double2* src, int64_t n, int ncols, double2* dst, cudaStream_t s);
void b_unpack(const double2* src, int64_t n, int ncols, double2* dst, cudaStream_t s);

}  // namespace pt
