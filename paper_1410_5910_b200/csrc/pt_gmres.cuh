// Device GMRES building blocks: CGS2 Arnoldi, Givens least squares, flags.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pt {

constexpr int RED_THREADS = 256;
constexpr int RED_BLOCKS = 296;  // fixed partial count => deterministic sums
constexpr int RED_CHUNK = 8;     // basis columns per pass of the dot kernel

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
  double2* V;         // n x (max_iter + 1), column j at V + j*n
  double2* P;         // RED_BLOCKS x ldp partials
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
};

// launch helpers (pt_gmres.cu); all stream-ordered, no host sync
void gm_dots(const double2* V, int64_t ldv, int ncols, const double2* w, int64_t n,
             double2* P, int ldp, int* nonfinite, cudaStream_t s);
void gm_reduce(const double2* P, int ldp, int ncols, double2* out, cudaStream_t s);
void gm_update_dots(const double2* V, int64_t ldv, int ncols, const double2* h, double2* w,
                    int64_t n, double2* P, int ldp, cudaStream_t s);
void gm_update_norm(const double2* V, int64_t ldv, int ncols, const double2* h, double2* w,
                    int64_t n, double2* P, int ldp, cudaStream_t s);
void gm_norm(const double2* w, int64_t n, double2* P, int ldp, int* nonfinite, cudaStream_t s);
void gm_begin(const GmresDev& g, cudaStream_t s);            // beta from hn2, g = beta e1
void gm_scale(double2* w, int64_t n, const DevStatus* st, int use_beta, cudaStream_t s);
void gm_givens(const GmresDev& g, int j, double rel_tol, int max_iter, const int* nonfinite,
               cudaStream_t s);
void gm_backsolve(const GmresDev& g, int k, cudaStream_t s);
void gm_combine(const double2* V, int64_t ldv, int k, const double2* y, double2* x, int64_t n,
                cudaStream_t s);
void gm_resid(const double2* b, const double2* ax, int64_t n, double2* P, int ldp,
              cudaStream_t s);
void gm_resid_finish(const GmresDev& g, cudaStream_t s);
void gm_zero(double2* x, int64_t n, cudaStream_t s);

}  // namespace pt
