// GMRES on the device: CGS2 Arnoldi + Givens least squares + report flags.
//
// Replaces gmres_solve (solver.py:231-295).  The reference orthogonalises
// with modified Gram-Schmidt (one pass, :259-261) and re-solves the
// Hessenberg least-squares problem with zgelsd every iteration (:269-272).
// Here: classical Gram-Schmidt with one re-orthogonalisation (CGS2), two
// passes of h = V^H w, w -= V h, and the Hessenberg is reduced by Givens
// rotations as it grows, so the relative residual |g_{j+1}| / beta falls
// out of one rotation instead of a least-squares solve.  The flag logic
// (breakdown, tolerance, stagnation window, maxiter) follows :265-289.
//
// Reductions are two-stage with a fixed number of partial blocks and a
// fixed summation order: repeat solves are bitwise identical.
#include <cmath>

#include "pt_device.cuh"
#include "pt_gmres.cuh"

namespace pt {

extern void count_launch();

namespace {

__device__ __forceinline__ void block_range(int64_t n, int64_t& lo, int64_t& hi) {
  const int64_t chunk = (n + RED_BLOCKS - 1) / RED_BLOCKS;
  lo = (int64_t)blockIdx.x * chunk;
  hi = lo + chunk < n ? lo + chunk : n;
}

// block-wide sum of RED_CHUNK complex values; thread u < RED_CHUNK returns sum u
__device__ void block_sum_chunk(double2 (&acc)[RED_CHUNK], double2 (*red)[RED_CHUNK],
                                double2* outp, int count) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int u = 0; u < RED_CHUNK; ++u) {
    const double2 v = warp_sum(acc[u]);
    if (lane == 0) red[warp][u] = v;
  }
  __syncthreads();
  if (threadIdx.x < count) {
    double2 s = make_double2(0.0, 0.0);
    for (int w = 0; w < RED_THREADS / 32; ++w) s = cadd(s, red[w][threadIdx.x]);
    outp[threadIdx.x] = s;
  }
  __syncthreads();
}

// P[b, i] = sum_{e in block b} conj(V_i[e]) w[e]
__device__ void dots_pass(const double2* V, int64_t ldv, int ncols, const double2* w,
                          int64_t lo, int64_t hi, double2* Prow) {
  __shared__ double2 red[RED_THREADS / 32][RED_CHUNK];
  for (int c0 = 0; c0 < ncols; c0 += RED_CHUNK) {
    double2 acc[RED_CHUNK];
#pragma unroll
    for (int u = 0; u < RED_CHUNK; ++u) acc[u] = make_double2(0.0, 0.0);
    const int cnt = ncols - c0 < RED_CHUNK ? ncols - c0 : RED_CHUNK;
    for (int64_t e = lo + threadIdx.x; e < hi; e += RED_THREADS) {
      const double2 wv = ld_cg(w + e);
#pragma unroll
      for (int u = 0; u < RED_CHUNK; ++u)
        if (u < cnt) acc[u] = cfma_conj(ld_cg(V + (int64_t)(c0 + u) * ldv + e), wv, acc[u]);
    }
    block_sum_chunk(acc, red, Prow + c0, cnt);
  }
}

__global__ void __launch_bounds__(RED_THREADS)
k_dots(const double2* V, int64_t ldv, int ncols, const double2* w, int64_t n, double2* P,
       int ldp, int* nonfinite) {
  int64_t lo, hi;
  block_range(n, lo, hi);
  if (nonfinite) {
    int bad = 0;
    for (int64_t e = lo + threadIdx.x; e < hi; e += RED_THREADS) {
      const double2 v = ld_cg(w + e);
      bad |= !(isfinite(v.x) && isfinite(v.y));
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
  }
  dots_pass(V, ldv, ncols, w, lo, hi, P + (int64_t)blockIdx.x * ldp);
}

// w -= V h, in place; own elements only
__device__ void update_pass(const double2* V, int64_t ldv, int ncols, const double2* hs,
                            double2* w, int64_t lo, int64_t hi) {
  for (int64_t e = lo + threadIdx.x; e < hi; e += RED_THREADS) {
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < ncols; ++i) acc = cfma(ld_cg(V + (int64_t)i * ldv + e), hs[i], acc);
    st_cg(w + e, csub(ld_cg(w + e), acc));
  }
}

__global__ void __launch_bounds__(RED_THREADS)
k_update_dots(const double2* V, int64_t ldv, int ncols, const double2* h, double2* w, int64_t n,
              double2* P, int ldp) {
  extern __shared__ double2 hs[];
  for (int i = threadIdx.x; i < ncols; i += RED_THREADS) hs[i] = h[i];
  __syncthreads();
  int64_t lo, hi;
  block_range(n, lo, hi);
  update_pass(V, ldv, ncols, hs, w, lo, hi);
  dots_pass(V, ldv, ncols, w, lo, hi, P + (int64_t)blockIdx.x * ldp);
}

__device__ void norm_pass(const double2* w, int64_t lo, int64_t hi, double2* outp) {
  __shared__ double2 red[RED_THREADS / 32][RED_CHUNK];
  double2 acc[RED_CHUNK];
#pragma unroll
  for (int u = 0; u < RED_CHUNK; ++u) acc[u] = make_double2(0.0, 0.0);
  for (int64_t e = lo + threadIdx.x; e < hi; e += RED_THREADS) {
    const double2 v = ld_cg(w + e);
    acc[0].x = fma(v.x, v.x, acc[0].x);
    acc[0].x = fma(v.y, v.y, acc[0].x);
  }
  block_sum_chunk(acc, red, outp, 1);
}

__global__ void __launch_bounds__(RED_THREADS)
k_update_norm(const double2* V, int64_t ldv, int ncols, const double2* h, double2* w, int64_t n,
              double2* P, int ldp) {
  extern __shared__ double2 hs[];
  for (int i = threadIdx.x; i < ncols; i += RED_THREADS) hs[i] = h[i];
  __syncthreads();
  int64_t lo, hi;
  block_range(n, lo, hi);
  update_pass(V, ldv, ncols, hs, w, lo, hi);
  norm_pass(w, lo, hi, P + (int64_t)blockIdx.x * ldp);
}

__global__ void __launch_bounds__(RED_THREADS)
k_norm(const double2* w, int64_t n, double2* P, int ldp, int* nonfinite) {
  int64_t lo, hi;
  block_range(n, lo, hi);
  if (nonfinite) {
    int bad = 0;
    for (int64_t e = lo + threadIdx.x; e < hi; e += RED_THREADS) {
      const double2 v = ld_cg(w + e);
      bad |= !(isfinite(v.x) && isfinite(v.y));
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
  }
  norm_pass(w, lo, hi, P + (int64_t)blockIdx.x * ldp);
}

// out[i] = sum_b P[b, i], fixed order
__global__ void k_reduce(const double2* P, int ldp, int ncols, double2* out) {
  for (int i = threadIdx.x; i < ncols; i += blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    for (int b = 0; b < RED_BLOCKS; ++b) s = cadd(s, P[(int64_t)b * ldp + i]);
    out[i] = s;
  }
}

__global__ void k_begin(GmresDev g) {
  DevStatus* st = g.st;
  const double beta = sqrt(g.hn2[0].x);
  st->iterations = 0;
  st->flag = 0;
  st->converged = 0;
  st->stop = 0;
  st->nonfinite = 0;
  st->breakdown = 0;
  st->rel = 1.0;
  st->beta = beta;
  st->inv_hn = beta > 0.0 ? 1.0 / beta : 0.0;
  st->hn = beta;
  for (int i = 0; i <= g.max_iter; ++i) g.g[i] = make_double2(0.0, 0.0);
  g.g[0] = make_double2(beta, 0.0);
}

__global__ void k_scale(double2* w, int64_t n, const DevStatus* st) {
  const double s = st->inv_hn;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double2 v = ld_cg(w + e);
    v.x *= s;
    v.y *= s;
    st_cg(w + e, v);
  }
}

__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }

// One Arnoldi column j: h = h1 + h2, hn = ||w||; rotations; flags.
__global__ void k_givens(GmresDev g, int j, double rel_tol, int max_iter,
                         const int* nonfinite) {
  DevStatus* st = g.st;
  if (*nonfinite) {
    st->nonfinite = 1;
    st->stop = 1;
    st->converged = 0;
    return;
  }
  const int ldr = g.max_iter + 1;
  double2* Rj = g.R + (int64_t)j * ldr;
  double2* Hj = g.Hraw + (int64_t)j * ldr;
  for (int i = 0; i <= j; ++i) {
    const double2 h = cadd(g.h1[i], g.h2[i]);
    Rj[i] = h;
    Hj[i] = h;
  }
  const double hn = sqrt(g.hn2[0].x);
  Hj[j + 1] = make_double2(hn, 0.0);
  // previous rotations
  for (int i = 0; i < j; ++i) {
    const double c = g.cs[i];
    const double2 s = g.sn[i];
    const double2 a = Rj[i], b = Rj[i + 1];
    Rj[i] = cadd(make_double2(c * a.x, c * a.y), cmul(s, b));
    const double2 sc = make_double2(-s.x, s.y);  // -conj(s)
    Rj[i + 1] = cadd(cmul(sc, a), make_double2(c * b.x, c * b.y));
  }
  // new rotation zeroing hn below Rj[j]
  const double2 a = Rj[j];
  const double aa = sqrt(cabs2(a));
  double c;
  double2 s, rr;
  if (aa == 0.0) {
    c = 0.0;
    s = make_double2(1.0, 0.0);
    rr = make_double2(hn, 0.0);
  } else {
    const double r = hypot(aa, hn);
    const double2 ph = make_double2(a.x / aa, a.y / aa);
    c = aa / r;
    s = make_double2(ph.x * hn / r, ph.y * hn / r);
    rr = make_double2(ph.x * r, ph.y * r);
  }
  if (aa == 0.0 && hn == 0.0) {
    c = 1.0;
    s = make_double2(0.0, 0.0);
    rr = make_double2(0.0, 0.0);
  }
  g.cs[j] = c;
  g.sn[j] = s;
  Rj[j] = rr;
  Rj[j + 1] = make_double2(0.0, 0.0);
  const double2 gj = g.g[j];
  g.g[j] = make_double2(c * gj.x, c * gj.y);
  g.g[j + 1] = cmul(make_double2(-s.x, s.y), gj);
  const double beta = st->beta;
  const double rel = sqrt(cabs2(g.g[j + 1])) / beta;
  g.hist[j] = rel;
  const int k = j + 1;
  st->iterations = k;
  st->rel = rel;
  st->hn = hn;
  const bool breakdown = hn <= BREAKDOWN_REL * beta;
  st->breakdown = breakdown ? 1 : 0;
  st->inv_hn = breakdown ? 0.0 : 1.0 / hn;
  if (breakdown) {
    st->converged = 1;
    st->flag = 1;  // breakdown
    st->stop = 1;
    return;
  }
  if (rel <= rel_tol) {
    st->converged = 1;
    st->flag = 0;
    st->stop = 1;
    return;
  }
  if (k > STAG_WINDOW) {
    const double old = g.hist[k - 1 - STAG_WINDOW];
    if (old > 0.0 && 1.0 - rel / old < STAG_IMPROVEMENT) {
      st->flag = 2;  // stagnation
      st->stop = 1;
      return;
    }
  }
  if (k >= max_iter) {
    st->flag = 3;  // maxiter
    st->stop = 1;
  }
}

// R y = g[0:k] (upper triangular k x k); a zero pivot gives y_i = 0
__global__ void k_backsolve(GmresDev g, int k) {
  const int ldr = g.max_iter + 1;
  for (int i = k - 1; i >= 0; --i) {
    double2 acc = g.g[i];
    for (int l = i + 1; l < k; ++l) acc = csub(acc, cmul(g.R[(int64_t)l * ldr + i], g.y[l]));
    const double2 d = g.R[(int64_t)i * ldr + i];
    const double dd = cabs2(d);
    if (dd == 0.0) {
      g.y[i] = make_double2(0.0, 0.0);
    } else {
      // acc / d
      g.y[i] = make_double2((acc.x * d.x + acc.y * d.y) / dd, (acc.y * d.x - acc.x * d.y) / dd);
    }
  }
}

__global__ void k_combine(const double2* V, int64_t ldv, int k, const double2* y, double2* x,
                          int64_t n) {
  extern __shared__ double2 ys[];
  for (int i = threadIdx.x; i < k; i += blockDim.x) ys[i] = y[i];
  __syncthreads();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < k; ++i) acc = cfma(ld_cg(V + (int64_t)i * ldv + e), ys[i], acc);
    st_cg(x + e, acc);
  }
}

__global__ void __launch_bounds__(RED_THREADS)
k_resid(const double2* b, const double2* ax, int64_t n, double2* P, int ldp) {
  __shared__ double2 red[RED_THREADS / 32][RED_CHUNK];
  int64_t lo, hi;
  block_range(n, lo, hi);
  double2 acc[RED_CHUNK];
#pragma unroll
  for (int u = 0; u < RED_CHUNK; ++u) acc[u] = make_double2(0.0, 0.0);
  for (int64_t e = lo + threadIdx.x; e < hi; e += RED_THREADS) {
    const double2 bv = ld_cg(b + e);
    const double2 r = csub(bv, ld_cg(ax + e));
    acc[0].x = fma(r.x, r.x, acc[0].x);
    acc[0].x = fma(r.y, r.y, acc[0].x);
    acc[1].x = fma(bv.x, bv.x, acc[1].x);
    acc[1].x = fma(bv.y, bv.y, acc[1].x);
  }
  block_sum_chunk(acc, red, P + (int64_t)blockIdx.x * ldp, 2);
}

__global__ void k_resid_finish(const double2* P, int ldp, DevStatus* st) {
  double a = 0.0, b = 0.0;
  for (int i = 0; i < RED_BLOCKS; ++i) {
    a += P[(int64_t)i * ldp].x;
    b += P[(int64_t)i * ldp + 1].x;
  }
  st->true_num2 = a;
  st->b_norm2 = b;
}

__global__ void k_zero(double2* x, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    x[e] = make_double2(0.0, 0.0);
}

int grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (int)(b < 1184 ? (b < 1 ? 1 : b) : 1184);
}

}  // namespace

void gm_dots(const double2* V, int64_t ldv, int ncols, const double2* w, int64_t n, double2* P,
             int ldp, int* nonfinite, cudaStream_t s) {
  count_launch();
  k_dots<<<RED_BLOCKS, RED_THREADS, 0, s>>>(V, ldv, ncols, w, n, P, ldp, nonfinite);
}
void gm_reduce(const double2* P, int ldp, int ncols, double2* out, cudaStream_t s) {
  count_launch();
  k_reduce<<<1, 128, 0, s>>>(P, ldp, ncols, out);
}
void gm_update_dots(const double2* V, int64_t ldv, int ncols, const double2* h, double2* w,
                    int64_t n, double2* P, int ldp, cudaStream_t s) {
  count_launch();
  k_update_dots<<<RED_BLOCKS, RED_THREADS, ncols * sizeof(double2), s>>>(V, ldv, ncols, h, w, n,
                                                                         P, ldp);
}
void gm_update_norm(const double2* V, int64_t ldv, int ncols, const double2* h, double2* w,
                    int64_t n, double2* P, int ldp, cudaStream_t s) {
  count_launch();
  k_update_norm<<<RED_BLOCKS, RED_THREADS, ncols * sizeof(double2), s>>>(V, ldv, ncols, h, w, n,
                                                                         P, ldp);
}
void gm_norm(const double2* w, int64_t n, double2* P, int ldp, int* nonfinite, cudaStream_t s) {
  count_launch();
  k_norm<<<RED_BLOCKS, RED_THREADS, 0, s>>>(w, n, P, ldp, nonfinite);
}
void gm_begin(const GmresDev& g, cudaStream_t s) {
  count_launch();
  k_begin<<<1, 1, 0, s>>>(g);
}
void gm_scale(double2* w, int64_t n, const DevStatus* st, int, cudaStream_t s) {
  count_launch();
  k_scale<<<grid_for(n), 256, 0, s>>>(w, n, st);
}
void gm_givens(const GmresDev& g, int j, double rel_tol, int max_iter, const int* nonfinite,
               cudaStream_t s) {
  count_launch();
  k_givens<<<1, 1, 0, s>>>(g, j, rel_tol, max_iter, nonfinite);
}
void gm_backsolve(const GmresDev& g, int k, cudaStream_t s) {
  count_launch();
  k_backsolve<<<1, 1, 0, s>>>(g, k);
}
void gm_combine(const double2* V, int64_t ldv, int k, const double2* y, double2* x, int64_t n,
                cudaStream_t s) {
  count_launch();
  k_combine<<<grid_for(n), 256, (k > 0 ? k : 1) * sizeof(double2), s>>>(V, ldv, k, y, x, n);
}
void gm_resid(const double2* b, const double2* ax, int64_t n, double2* P, int ldp,
              cudaStream_t s) {
  count_launch();
  k_resid<<<RED_BLOCKS, RED_THREADS, 0, s>>>(b, ax, n, P, ldp);
}
void gm_resid_finish(const GmresDev& g, cudaStream_t s) {
  count_launch();
  k_resid_finish<<<1, 1, 0, s>>>(g.P, g.ldp, g.st);
}
void gm_zero(double2* x, int64_t n, cudaStream_t s) {
  count_launch();
  k_zero<<<grid_for(n), 256, 0, s>>>(x, n);
}

}  // namespace pt
