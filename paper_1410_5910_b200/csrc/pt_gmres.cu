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
// Each Arnoldi step is four kernels.  Block partial sums are reduced by the
// last block to finish (ticket counter), always over all blocks in index
// order, so results are bitwise repeatable.  Every step kernel returns at
// once when the status says the solve has stopped: the host enqueues steps
// ahead of its convergence check without changing the result.
#include <cmath>

#include "pt_device.cuh"
#include "pt_gmres.cuh"

namespace pt {

extern void count_launch();

namespace {

__device__ __forceinline__ bool stopped(const DevStatus* st) {
  return *((volatile const int*)&st->stop) != 0;
}

__device__ __forceinline__ void block_range(int64_t n, int64_t& lo, int64_t& hi) {
  const int64_t chunk = (n + RED_BLOCKS - 1) / RED_BLOCKS;
  lo = (int64_t)blockIdx.x * chunk;
  hi = lo + chunk < n ? lo + chunk : n;
}

// block-wide sum of RED_CHUNK complex values; thread u < count writes sum u
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
    st_cg(outp + threadIdx.x, s);
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

// w -= V hs, in place; own elements only
__device__ void update_pass(const double2* V, int64_t ldv, int ncols, const double2* hs,
                            double2* w, int64_t lo, int64_t hi) {
  for (int64_t e = lo + threadIdx.x; e < hi; e += RED_THREADS) {
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < ncols; ++i) acc = cfma(ld_cg(V + (int64_t)i * ldv + e), hs[i], acc);
    st_cg(w + e, csub(ld_cg(w + e), acc));
  }
}

// The last block to arrive sums the partials of all blocks (index order).
__device__ bool last_block(int* ticket) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (s_last) __threadfence();
  return s_last != 0;
}

__device__ void reduce_partials(const double2* P, int ldp, int ncols, double2* out) {
  for (int i = threadIdx.x; i < ncols; i += blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    for (int b = 0; b < RED_BLOCKS; ++b) s = cadd(s, ld_cg(P + (int64_t)b * ldp + i));
    st_cg(out + i, s);
  }
}

__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }

// Arnoldi column j: h = h1 + h2, hn; rotations; residual; flags (one thread)
__device__ void givens_update(const GmresDev& g, int j, double rel_tol, int max_iter) {
  DevStatus* st = g.st;
  if (*((volatile int*)g.nonfinite)) {
    st->nonfinite = 1;
    st->stop = 1;
    st->converged = 0;
    return;
  }
  const int ldr = g.max_iter + 1;
  double2* Rj = g.R + (int64_t)j * ldr;
  double2* Hj = g.Hraw + (int64_t)j * ldr;
  for (int i = 0; i <= j; ++i) {
    const double2 h = cadd(ld_cg(g.h1 + i), ld_cg(g.h2 + i));
    Rj[i] = h;
    Hj[i] = h;
  }
  const double hn = sqrt(ld_cg(g.hn2).x);
  Hj[j + 1] = make_double2(hn, 0.0);
  for (int i = 0; i < j; ++i) {
    const double c = g.cs[i];
    const double2 s = g.sn[i];
    const double2 a = Rj[i], b = Rj[i + 1];
    Rj[i] = cadd(make_double2(c * a.x, c * a.y), cmul(s, b));
    Rj[i + 1] = cadd(cmul(make_double2(-s.x, s.y), a), make_double2(c * b.x, c * b.y));
  }
  // rotation zeroing hn below Rj[j]:  [c s; -conj(s) c] [a; hn] = [r; 0]
  const double2 a = Rj[j];
  const double aa = sqrt(cabs2(a));
  double c;
  double2 s, rr;
  if (aa == 0.0 && hn == 0.0) {
    c = 1.0;
    s = make_double2(0.0, 0.0);
    rr = make_double2(0.0, 0.0);
  } else if (aa == 0.0) {
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
  const bool breakdown = hn <= BREAKDOWN_REL * beta;  // solver.py:265
  st->breakdown = breakdown ? 1 : 0;
  st->inv_hn = breakdown ? 0.0 : 1.0 / hn;
  if (breakdown) {
    st->converged = 1;
    st->flag = 1;
    st->stop = 1;
  } else if (rel <= rel_tol) {  // solver.py:279
    st->converged = 1;
    st->flag = 0;
    st->stop = 1;
  } else if (k > STAG_WINDOW &&  // solver.py:282-287
             g.hist[k - 1 - STAG_WINDOW] > 0.0 &&
             1.0 - rel / g.hist[k - 1 - STAG_WINDOW] < STAG_IMPROVEMENT) {
    st->flag = 2;
    st->stop = 1;
  } else if (k >= max_iter) {  // for/else, solver.py:288-289
    st->flag = 3;
    st->stop = 1;
  }
  __threadfence();
}

// ---- kernels -----------------------------------------------------------------

__global__ void __launch_bounds__(RED_THREADS) k_h1(GmresDev g) {
  if (stopped(g.st)) return;
  const int j = g.st->iterations;
  const double2* w = g.V + (int64_t)(j + 1) * g.n;
  int64_t lo, hi;
  block_range(g.n, lo, hi);
  int bad = 0;
  for (int64_t e = lo + threadIdx.x; e < hi; e += RED_THREADS) {
    const double2 v = ld_cg(w + e);
    bad |= !(isfinite(v.x) && isfinite(v.y));
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(g.nonfinite, 1);
  dots_pass(g.V, g.n, j + 1, w, lo, hi, g.P + (int64_t)blockIdx.x * g.ldp);
  if (last_block(g.ticket + 0)) {
    reduce_partials(g.P, g.ldp, j + 1, g.h1);
    if (threadIdx.x == 0) g.ticket[0] = 0;
  }
}

__global__ void __launch_bounds__(RED_THREADS) k_h2(GmresDev g) {
  if (stopped(g.st)) return;
  const int j = g.st->iterations;
  extern __shared__ double2 hs[];
  const int nc = j + 1;
  for (int i = threadIdx.x; i < nc; i += RED_THREADS) hs[i] = ld_cg(g.h1 + i);
  __syncthreads();
  double2* w = g.V + (int64_t)(j + 1) * g.n;
  int64_t lo, hi;
  block_range(g.n, lo, hi);
  update_pass(g.V, g.n, nc, hs, w, lo, hi);
  dots_pass(g.V, g.n, nc, w, lo, hi, g.P + (int64_t)blockIdx.x * g.ldp);
  if (last_block(g.ticket + 1)) {
    reduce_partials(g.P, g.ldp, nc, g.h2);
    if (threadIdx.x == 0) g.ticket[1] = 0;
  }
}

__global__ void __launch_bounds__(RED_THREADS)
k_norm_givens(GmresDev g, double rel_tol, int max_iter, cudaGraphConditionalHandle cond) {
  if (stopped(g.st)) return;
  const int j = g.st->iterations;
  extern __shared__ double2 hs[];
  const int nc = j + 1;
  for (int i = threadIdx.x; i < nc; i += RED_THREADS) hs[i] = ld_cg(g.h2 + i);
  __syncthreads();
  double2* w = g.V + (int64_t)(j + 1) * g.n;
  int64_t lo, hi;
  block_range(g.n, lo, hi);
  update_pass(g.V, g.n, nc, hs, w, lo, hi);
  norm_pass(w, lo, hi, g.P + (int64_t)blockIdx.x * g.ldp);
  if (last_block(g.ticket + 2)) {
    reduce_partials(g.P, g.ldp, 1, g.hn2);
    __syncthreads();
    __threadfence_block();
    if (threadIdx.x == 0) {
      g.ticket[2] = 0;
      givens_update(g, j, rel_tol, max_iter);
      if (cond) cudaGraphSetConditional(cond, g.st->stop ? 0u : 1u);
    }
  }
}

// v_{j+1} = w / ||w||; skipped once the solve stopped (column k is unused)
__global__ void k_normalize(GmresDev g) {
  const DevStatus* st = g.st;
  if (stopped(st)) return;
  const double s = st->inv_hn;
  double2* w = g.V + (int64_t)st->iterations * g.n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < g.n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double2 v = ld_cg(w + e);
    v.x *= s;
    v.y *= s;
    st_cg(w + e, v);
  }
}

__global__ void __launch_bounds__(RED_THREADS)
k_begin_norm(GmresDev g, cudaGraphConditionalHandle cond) {
  int64_t lo, hi;
  block_range(g.n, lo, hi);
  norm_pass(g.V, lo, hi, g.P + (int64_t)blockIdx.x * g.ldp);
  if (last_block(g.ticket + 0)) {
    reduce_partials(g.P, g.ldp, 1, g.hn2);
    __syncthreads();
    __threadfence_block();
    if (threadIdx.x == 0) {
      g.ticket[0] = 0;
      DevStatus* st = g.st;
      const double beta = sqrt(ld_cg(g.hn2).x);
      st->iterations = 0;
      st->flag = 0;
      st->converged = 0;
      st->nonfinite = 0;
      st->breakdown = 0;
      st->rel = 1.0;
      st->beta = beta;
      st->inv_hn = beta > 0.0 ? 1.0 / beta : 0.0;
      st->hn = beta;
      *g.nonfinite = 0;
      for (int i = 0; i <= g.max_iter; ++i) g.g[i] = make_double2(0.0, 0.0);
      g.g[0] = make_double2(beta, 0.0);
      // beta == 0: x = 0, converged (solver.py:239-242)
      st->converged = beta == 0.0 ? 1 : 0;
      st->stop = beta == 0.0 ? 1 : 0;
      __threadfence();
      if (cond) cudaGraphSetConditional(cond, beta == 0.0 ? 0u : 1u);
    }
  }
}

__global__ void k_begin_scale(GmresDev g) {
  const double s = g.st->inv_hn;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < g.n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double2 v = ld_cg(g.V + e);
    v.x *= s;
    v.y *= s;
    st_cg(g.V + e, v);
  }
}

// R y = g[0:k] (upper triangular k x k, k = iterations); a zero pivot gives y_i = 0
__global__ void k_backsolve(GmresDev g) {
  const int k = g.st->iterations;
  const int ldr = g.max_iter + 1;
  for (int i = k - 1; i >= 0; --i) {
    double2 acc = g.g[i];
    for (int l = i + 1; l < k; ++l) acc = csub(acc, cmul(g.R[(int64_t)l * ldr + i], g.y[l]));
    const double2 d = g.R[(int64_t)i * ldr + i];
    const double dd = cabs2(d);
    g.y[i] = dd == 0.0 ? make_double2(0.0, 0.0)
                       : make_double2((acc.x * d.x + acc.y * d.y) / dd,
                                      (acc.y * d.x - acc.x * d.y) / dd);
  }
}

// x = V[:, :k] y
__global__ void k_combine(GmresDev g, double2* x) {
  extern __shared__ double2 ys[];
  const int k = g.st->iterations;
  const double2* V = g.V;
  const double2* y = g.y;
  const int64_t ldv = g.n, n = g.n;
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
k_resid(GmresDev g, const double2* b, const double2* ax) {
  __shared__ double2 red[RED_THREADS / 32][RED_CHUNK];
  int64_t lo, hi;
  block_range(g.n, lo, hi);
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
  block_sum_chunk(acc, red, g.P + (int64_t)blockIdx.x * g.ldp, 2);
  if (last_block(g.ticket + 0)) {
    if (threadIdx.x == 0) {
      g.ticket[0] = 0;
      double a = 0.0, c = 0.0;
      for (int i = 0; i < RED_BLOCKS; ++i) {
        a += ld_cg(g.P + (int64_t)i * g.ldp).x;
        c += ld_cg(g.P + (int64_t)i * g.ldp + 1).x;
      }
      g.st->true_num2 = a;
      g.st->b_norm2 = c;
    }
  }
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

void gm_arnoldi_step(const GmresDev& g, double rel_tol, int max_iter,
                     cudaGraphConditionalHandle cond, cudaStream_t s) {
  const size_t hs = (size_t)(g.max_iter + 1) * sizeof(double2);
  count_launch();
  k_h1<<<RED_BLOCKS, RED_THREADS, 0, s>>>(g);
  count_launch();
  k_h2<<<RED_BLOCKS, RED_THREADS, hs, s>>>(g);
  count_launch();
  k_norm_givens<<<RED_BLOCKS, RED_THREADS, hs, s>>>(g, rel_tol, max_iter, cond);
  count_launch();
  k_normalize<<<grid_for(g.n), 256, 0, s>>>(g);
}

void gm_begin(const GmresDev& g, cudaGraphConditionalHandle cond, cudaStream_t s) {
  count_launch();
  k_begin_norm<<<RED_BLOCKS, RED_THREADS, 0, s>>>(g, cond);
  count_launch();
  k_begin_scale<<<grid_for(g.n), 256, 0, s>>>(g);
}

void gm_finish(const GmresDev& g, double2* x, cudaStream_t s) {
  count_launch();
  k_backsolve<<<1, 1, 0, s>>>(g);
  count_launch();
  k_combine<<<grid_for(g.n), 256, (size_t)(g.max_iter + 1) * sizeof(double2), s>>>(g, x);
}

void gm_resid(const GmresDev& g, const double2* b, const double2* ax, cudaStream_t s) {
  count_launch();
  k_resid<<<RED_BLOCKS, RED_THREADS, 0, s>>>(g, b, ax);
}

void gm_zero(double2* x, int64_t n, cudaStream_t s) {
  count_launch();
  k_zero<<<grid_for(n), 256, 0, s>>>(x, n);
}

}  // namespace pt
