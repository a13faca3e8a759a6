// Device GMRES building blocks: CGS2 Arnoldi, Givens least squares, flags.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pt {

constexpr int RED_THREADS = 256;
constexpr int RED_BLOCKS = 296;  // fixed partial count => deterministic sums
constexpr int RED_CHUNK = 8;     // basis columns per pass of the dot kernel
constexpr int ARN_THREADS = 512; // fused Arnoldi step: threads per block
constexpr int ARN_MAX_BLOCKS = RED_BLOCKS;
constexpr int ARN_SMEM_VECS = 5;   // Arnoldi step: coefficients + Givens operands (ldp each)

// STAGNATION_WINDOW / STAGNATION_IMPROVEMENT of solver.py:55-56
constexpr int STAG_WINDOW = 10;
constexpr double STAG_IMPROVEMENT = 1e-3;
constexpr double BREAKDOWN_REL = 1e-14;  // solver.py:265

struct DevStatus {
  int iterations;
  int flag;
  int converged;
  int stop;
  int nonfinite;
  int breakdown;
  double rel;
  double beta;
  double inv_hn;
  double hn;
  double true_num2;   // ||b - A x||^2
  double b_norm2;     // ||b||^2
};

struct GmresDev {
  int64_t n;
  int max_iter;
  int ldp;            // partial row stride (>= max_iter + 2)
  int arn_blocks;     // blocks of the fused Arnoldi step (one per SM, co-resident)
  int64_t arn_vcap;   // complex elements of a block's staged V slice
  double2* V;         // n x (max_iter + 1), column j at V + j*n
  double2* P;         // 2 x RED_BLOCKS x ldp partials
  double2* h1;        // CGS pass 1 coefficients
  double2* h2;        // CGS pass 2 coefficients
  double2* hn2;       // [0].x = ||w||^2
  double2* R;         // rotated Hessenberg, column-major (max_iter+1) x max_iter
  double2* Hraw;      // raw Hessenberg (record)
  double2* g;         // rotated rhs, max_iter + 1
  double* cs;         // rotation cosines
  double2* sn;        // rotation sines
  double* hist;       // residual history
  double2* y;         // least-squares solution
  DevStatus* st;
  int* ticket;        // last-block tickets of the fused reductions (3)
  int* nonfinite;
};

// launch helpers (pt_gmres.cu); all stream-ordered and graph-capturable.
// The iteration index j is read on the device (st->iterations), and every
// iteration kernel returns at once when st->stop is set, so the same
// kernels serve the per-step API, a speculative host loop and the CUDA
// graph whose conditional WHILE node runs the whole loop on the device
// (cond != 0: the kernels set the loop condition).
// One Arnoldi step (w = basis column j+1):
//   h1 = V^H w (+ non-finite check) | w -= V h1, h2 = V^H w |
//   w -= V h2, ||w||, Givens + flags | w /= ||w||
// One cooperative kernel (grid-wide barriers between the reductions).
cudaError_t gm_arnoldi_step(const GmresDev& g, double rel_tol, int max_iter,
                            cudaGraphConditionalHandle cond, cudaStream_t s);
// blocks / shared memory of the fused step for this workspace (once)
cudaError_t gm_arnoldi_setup(GmresDev& g, int device);
// ||V0||, beta, g = beta e1, V0 /= beta; stop if beta == 0
void gm_begin(const GmresDev& g, cudaGraphConditionalHandle cond, cudaStream_t s);
// y = R^-1 g, x = V[:, :k] y (k = st->iterations)
void gm_finish(const GmresDev& g, double2* x, cudaStream_t s);
void gm_resid(const GmresDev& g, const double2* b, const double2* ax, cudaStream_t s);
void gm_zero(double2* x, int64_t n, cudaStream_t s);

}  // namespace pt
