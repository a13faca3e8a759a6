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
// Each Arnoldi step is one cooperative kernel, one block per SM, with three
// grid-wide barriers (after h1, h2 and ||w|| partials).  Every block reduces
// the block partials itself in the same fixed order, so all blocks hold the
// same coefficients and results are bitwise repeatable.  The begin / finish
// kernels reduce partials in the last block to finish (ticket counter).  Every step kernel returns at
// once when the status says the solve has stopped: the host enqueues steps
// ahead of its convergence check without changing the result.
#ifdef PT_ARN_PROFILE
#include <cstdlib>
#include <cstdio>
#endif
#include <cooperative_groups.h>

#include <algorithm>
#include <atomic>
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

// out[c] = sum of the RED_BLOCKS partials P[b, c] (c < ncols): every thread
// sums a fixed strided subset, then a fixed tree over the block -- all loads
// in flight at once (a serial sum is one L2 round trip per partial)
__device__ void reduce_partials(const double2* P, int ldp, int ncols, double2* out) {
  __shared__ double2 red[RED_THREADS / 32];
  for (int c = 0; c < ncols; ++c) {
    double2 s = make_double2(0.0, 0.0);
    for (int b = threadIdx.x; b < RED_BLOCKS; b += RED_THREADS)
      s = cadd(s, ld_cg(P + (int64_t)b * ldp + c));
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double2 t = make_double2(0.0, 0.0);
      for (int w = 0; w < RED_THREADS / 32; ++w) t = cadd(t, red[w]);
      st_cg(out + c, t);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }

// Operands of the Givens update, gathered into shared memory by block 0 of
// the Arnoldi step while the reductions run: the one-thread rotation chain
// then reads no global memory (a global load per rotation, ordered behind
// the previous rotation's stores, cost ~0.4 us each: 14 us at j = 35).
// Dynamic shared memory of the step: [coefficients | h1 | h2 | cs (.x) | sn]
// (ldp complex values each; h1/h2 = CGS pass 1/2 coefficients of rows 0..j,
// cs/sn = rotations 0..j-1), then the block's slice of w and of V.
struct GivensSmem {
  double2 gj;   // g[j]
  double beta;
  double hist_w;  // hist[k - 1 - STAG_WINDOW] (k > STAG_WINDOW)
  int nonfinite;
};

// Arnoldi column j: h = h1 + h2, hn; rotations; residual; flags (one thread)
__device__ __noinline__ void givens_update(const GmresDev& g, const GivensSmem& q, int j, double hn,
                              double rel_tol, int max_iter) {
  DevStatus* st = g.st;
  if (q.nonfinite) {
    st->nonfinite = 1;
    st->stop = 1;
    st->converged = 0;
    return;
  }
  const int ldr = g.max_iter + 1;
  double2* Rj = g.R + (int64_t)j * ldr;
  double2* Hj = g.Hraw + (int64_t)j * ldr;
  Hj[j + 1] = make_double2(hn, 0.0);
  // previous rotations down the new column; the running entry is carried in
  // registers, the operands come from shared memory (indexed off the
  // dynamic shared-memory symbol, so the compiler knows they cannot alias
  // the global stores and issues them ahead of the rotation chain)
  extern __shared__ double2 gsm[];
  const double2* h1 = gsm + g.ldp;
  const double2* h2 = gsm + 2 * g.ldp;
  const double2* cs = gsm + 3 * g.ldp;
  const double2* sn = gsm + 4 * g.ldp;
  double2 a = cadd(h1[0], h2[0]);
  Hj[0] = a;
#pragma unroll 4
  for (int i = 0; i < j; ++i) {
    const double2 b = cadd(h1[i + 1], h2[i + 1]);
    Hj[i + 1] = b;
    const double c = cs[i].x;
    const double2 s = sn[i];
    Rj[i] = cadd(make_double2(c * a.x, c * a.y), cmul(s, b));
    a = cadd(cmul(make_double2(-s.x, s.y), a), make_double2(c * b.x, c * b.y));
  }
  // rotation zeroing hn below Rj[j]:  [c s; -conj(s) c] [a; hn] = [r; 0]
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
  const double2 gj = q.gj;
  const double2 gj1 = cmul(make_double2(-s.x, s.y), gj);
  g.g[j] = make_double2(c * gj.x, c * gj.y);
  g.g[j + 1] = gj1;
  const double beta = q.beta;
  const double rel = sqrt(cabs2(gj1)) / beta;
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
             q.hist_w > 0.0 && 1.0 - rel / q.hist_w < STAG_IMPROVEMENT) {
    st->flag = 2;
    st->stop = 1;
  } else if (k >= max_iter) {  // for/else, solver.py:288-289
    st->flag = 3;
    st->stop = 1;
  }
}

// ---- fused Arnoldi step ---------------------------------------------------------

// phase timestamps of the Arnoldi step (profiling build only: -DPT_ARN_PROFILE,
// tools/arn_phases.sh); block 0 and the last block print the phase deltas
#ifdef PT_ARN_PROFILE
#define ARN_MARK(i) \
  do {                                                                        \
    if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm[i])); \
  } while (0)
#else
#define ARN_MARK(i) \
  do {            \
  } while (0)
#endif

namespace cg = cooperative_groups;

// Partials of the Arnoldi step are stored column-major: the block-b partial
// of coefficient c is P[c * RED_BLOCKS + b], so the partials of one
// coefficient are contiguous and a warp reads them with coalesced loads
// (every block reads every partial: with a row-per-block layout the 148
// blocks' strided loads queued ~8x more L2 requests on the same lines, and
// the reduction took 6.8 us at j = 35).
//
// out[c] = sum over blocks b of the partials of c, c < nc: a warp per
// coefficient, lane l sums partials b = l, l + 32, ... in order (all loads
// issued before the adds), then a fixed xor tree -- the same result in every
// block
__device__ void arn_reduce(const double2* P, int nblk, int nc, double2* out) {
  constexpr int PER = (ARN_MAX_BLOCKS + 31) / 32;
  const int lane = threadIdx.x & 31;
  for (int c = (int)threadIdx.x >> 5; c < nc; c += ARN_THREADS / 32) {
    double2 v[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int b = lane + 32 * i;
      v[i] = b < nblk ? ld_cg(P + (int64_t)c * RED_BLOCKS + b) : make_double2(0.0, 0.0);
    }
    double2 s = v[0];
#pragma unroll
    for (int i = 1; i < PER; ++i) s = cadd(s, v[i]);
    s = warp_sum(s);
    if (lane == 0) out[c] = s;
  }
}

// P[blockIdx.x, c] = sum_{e in slice} conj(V_c[e]) w[e]; warp per column,
// the block's slice of w in shared memory; Vb = element 0 of the slice of
// column 0, columns ldb apart (global memory, or the slice staged in smem)
__device__ void arn_dots(const double2* Vb, int64_t ldb, int nc, const double2* ws, int len,
                         double2* P) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < nc; c += ARN_THREADS / 32) {
    const double2* v = Vb + (int64_t)c * ldb;
    // two accumulators (fixed assignment: elements e < len alternate), so the
    // FP64 FMA latency chain is half as long
    double2 a0 = make_double2(0.0, 0.0), a1 = a0;
    int e = lane;
    for (; e + 32 < len; e += 64) {  // generic: smem or global
      a0 = cfma_conj(v[e], ws[e], a0);
      a1 = cfma_conj(v[e + 32], ws[e + 32], a1);
    }
    if (e < len) a0 = cfma_conj(v[e], ws[e], a0);
    double2 acc = warp_sum(cadd(a0, a1));
    if (lane == 0) st_cg(P + (int64_t)c * RED_BLOCKS + blockIdx.x, acc);
  }
}

// ws[e] -= sum_c V_c[e] h[c] over the block's slice (thread per element)
__device__ void arn_update(const double2* Vb, int64_t ldb, int nc, const double2* h, double2* ws,
                           int len) {
  for (int e = threadIdx.x; e < len; e += ARN_THREADS) {
    // four accumulators over c mod 4 (fixed order of the final sum): the FP64
    // FMA latency chain is a quarter as long
    double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0;
    int c = 0;
    for (; c + 4 <= nc; c += 4) {
      a0 = cfma(Vb[(int64_t)c * ldb + e], h[c], a0);
      a1 = cfma(Vb[(int64_t)(c + 1) * ldb + e], h[c + 1], a1);
      a2 = cfma(Vb[(int64_t)(c + 2) * ldb + e], h[c + 2], a2);
      a3 = cfma(Vb[(int64_t)(c + 3) * ldb + e], h[c + 3], a3);
    }
    for (; c < nc; ++c) a0 = cfma(Vb[(int64_t)c * ldb + e], h[c], a0);
    ws[e] = csub(ws[e], cadd(cadd(a0, a1), cadd(a2, a3)));
  }
}

// w = basis column j+1 (written by the preconditioned matvec): CGS2 against
// columns 0..j, ||w||, Givens + flags (block 0), w /= ||w|| (every block).
__global__ void __launch_bounds__(ARN_THREADS, 1)
k_arnoldi(GmresDev g, double rel_tol, int max_iter, cudaGraphConditionalHandle cond) {
  extern __shared__ double2 sm[];
  if (stopped(g.st)) return;  // uniform: no block reaches a grid barrier
#ifdef PT_ARN_PROFILE
  unsigned long long tm[12] = {0};
#endif
  ARN_MARK(0);
  cg::grid_group grid = cg::this_grid();
  const int j = g.st->iterations;
  const int nc = j + 1;
  const int nblk = gridDim.x;
  const int64_t chunk = (g.n + nblk - 1) / nblk;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int len = (int)(lo + chunk < g.n ? chunk : (lo < g.n ? g.n - lo : 0));
  double2* hsm = sm;                  // coefficients (ldp)
  __shared__ GivensSmem gq;           // block 0: the Givens update's scalar operands
  double2* ws = sm + ARN_SMEM_VECS * g.ldp;  // the block's slice of w
  double2* vs = ws + chunk;           // the block's slice of V[:, 0..j] (when it fits)
  double2* w = g.V + (int64_t)(j + 1) * g.n;
  double2* P1 = g.P;
  double2* P2 = g.P + (int64_t)RED_BLOCKS * g.ldp;
  __shared__ int s_bad;
  __shared__ __align__(8) unsigned long long s_vbar;
  // the four passes over V read the block's slice once from HBM: staged in
  // shared memory with TMA bulk copies (one per column) when it fits
  const bool staged = (int64_t)nc * len <= g.arn_vcap && len > 0;
  const double2* Vb = staged ? vs : g.V + lo;
  const int64_t ldb = staged ? len : g.n;
  if (threadIdx.x == 0) {
    s_bad = 0;
    if (staged) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&s_vbar))
                   : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&s_vbar)),
                   "r"((uint32_t)(nc * len * sizeof(double2)))
                   : "memory");
    }
  }
  __syncthreads();
  if (staged)
    for (int c = threadIdx.x; c < nc; c += ARN_THREADS)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];" ::"r"((uint32_t)__cvta_generic_to_shared(vs + (int64_t)c * len)),
          "l"(g.V + (int64_t)c * g.n + lo), "r"((uint32_t)(len * sizeof(double2))),
          "r"((uint32_t)__cvta_generic_to_shared(&s_vbar))
          : "memory");
  if (blockIdx.x == 0) {  // Givens operands from earlier iterations (off the critical path)
    for (int i = threadIdx.x; i < j; i += ARN_THREADS) {
      sm[3 * g.ldp + i] = make_double2(g.cs[i], 0.0);
      sm[4 * g.ldp + i] = g.sn[i];
    }
    if (threadIdx.x == 32) {
      gq.gj = g.g[j];
      gq.beta = g.st->beta;
      gq.hist_w = j + 1 > STAG_WINDOW ? g.hist[j - STAG_WINDOW] : 0.0;
    }
  }
  int bad = 0;
  for (int e = threadIdx.x; e < len; e += ARN_THREADS) {
    const double2 v = ld_cg(w + lo + e);
    bad |= !(isfinite(v.x) && isfinite(v.y));
    ws[e] = v;
  }
  if (bad) atomicOr(&s_bad, 1);
  __syncthreads();
  if (s_bad && threadIdx.x == 0) atomicOr(g.nonfinite, 1);
  if (staged) {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
          " selp.u32 %0, 1, 0, p;\n}"
          : "=r"(done)
          : "r"((uint32_t)__cvta_generic_to_shared(&s_vbar))
          : "memory");
  }
  ARN_MARK(1);
  // pass 1: h1 = V^H w
  arn_dots(Vb, ldb, nc, ws, len, P1);
  ARN_MARK(2);
  grid.sync();
  ARN_MARK(3);
  // every block's non-finite flag is set before the first barrier
  if (blockIdx.x == 0 && threadIdx.x == 32) gq.nonfinite = *((volatile int*)g.nonfinite);
  arn_reduce(P1, nblk, nc, hsm);
  __syncthreads();
  if (blockIdx.x == 0)
    for (int c = threadIdx.x; c < nc; c += ARN_THREADS) {
      st_cg(g.h1 + c, hsm[c]);
      sm[g.ldp + c] = hsm[c];
    }
  __syncthreads();
  ARN_MARK(10);
  // pass 2: w -= V h1, h2 = V^H w
  arn_update(Vb, ldb, nc, hsm, ws, len);
  __syncthreads();
  ARN_MARK(11);
  arn_dots(Vb, ldb, nc, ws, len, P2);
  ARN_MARK(4);
  grid.sync();
  ARN_MARK(5);
  arn_reduce(P2, nblk, nc, hsm);
  __syncthreads();
  if (blockIdx.x == 0)
    for (int c = threadIdx.x; c < nc; c += ARN_THREADS) {
      st_cg(g.h2 + c, hsm[c]);
      sm[2 * g.ldp + c] = hsm[c];
    }
  __syncthreads();
  // w -= V h2, ||w||^2
  arn_update(Vb, ldb, nc, hsm, ws, len);
  {
    double2 acc = make_double2(0.0, 0.0);
    for (int e = threadIdx.x; e < len; e += ARN_THREADS) {
      const double2 v = ws[e];
      acc.x = fma(v.x, v.x, acc.x);
      acc.x = fma(v.y, v.y, acc.x);
    }
    __shared__ double2 red[ARN_THREADS / 32];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double2 s = make_double2(0.0, 0.0);
      for (int i = 0; i < ARN_THREADS / 32; ++i) s = cadd(s, red[i]);
      st_cg(P1 + blockIdx.x, s);  // P1 is free: pass-1 partials consumed
    }
  }
  ARN_MARK(6);
  grid.sync();
  ARN_MARK(7);
  arn_reduce(P1, nblk, 1, hsm);
  __syncthreads();
  const double hn = sqrt(hsm[0].x);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st_cg(g.hn2, hsm[0]);
    givens_update(g, gq, j, hn, rel_tol, max_iter);
    if (cond) cudaGraphSetConditional(cond, g.st->stop ? 0u : 1u);
  }
  ARN_MARK(8);
  // v_{j+1} = w / ||w|| (unused when the solve stops here; breakdown => 0)
  const double inv = hn <= BREAKDOWN_REL * g.st->beta ? 0.0 : 1.0 / hn;
  for (int e = threadIdx.x; e < len; e += ARN_THREADS) {
    double2 v = ws[e];
    v.x *= inv;
    v.y *= inv;
    st_cg(w + lo + e, v);
  }
  ARN_MARK(9);
#ifdef PT_ARN_PROFILE
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
    printf("ARN j=%d blk=%d stage %llu dots1 %llu sync1 %llu red+upd+dots2 %llu sync2 %llu "
           "red+upd+norm %llu sync3 %llu red+givens %llu normalize %llu total %llu [red1 %llu upd1 %llu]\n",
           j, blockIdx.x, tm[1] - tm[0], tm[2] - tm[1], tm[3] - tm[2], tm[4] - tm[3],
           tm[5] - tm[4], tm[6] - tm[5], tm[7] - tm[6], tm[8] - tm[7], tm[9] - tm[8],
           tm[9] - tm[0], tm[10] - tm[3], tm[11] - tm[10]);
#endif
}

// ---- kernels -----------------------------------------------------------------

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

// R y = g[0:k] (upper triangular k x k, k = iterations); a zero pivot gives
// y_i = 0.  One block: R and g in shared memory, column-oriented substitution
// (y_i, then every g_t, t < i, updated in parallel): k barrier steps instead
// of k^2 dependent global loads.
__global__ void __launch_bounds__(RED_THREADS) k_backsolve(GmresDev g) {
  extern __shared__ double2 rs[];  // k x k (column-major) + g
  const int k = g.st->iterations;
  const int ldr = g.max_iter + 1;
  double2* gs = rs + (int64_t)k * k;
  for (int i = threadIdx.x; i < k * k; i += blockDim.x)
    rs[i] = g.R[(int64_t)(i / k) * ldr + (i % k)];
  for (int i = threadIdx.x; i < k; i += blockDim.x) gs[i] = g.g[i];
  __syncthreads();
  for (int i = k - 1; i >= 0; --i) {
    const double2 d = rs[(int64_t)i * k + i];
    const double dd = d.x * d.x + d.y * d.y;
    const double2 acc = gs[i];
    const double2 yi = dd == 0.0 ? make_double2(0.0, 0.0)
                                 : make_double2((acc.x * d.x + acc.y * d.y) / dd,
                                                (acc.y * d.x - acc.x * d.y) / dd);
    __syncthreads();  // every thread has read gs[i]
    if (threadIdx.x == 0) g.y[i] = yi;
    for (int t = threadIdx.x; t < i; t += blockDim.x)
      gs[t] = csub(gs[t], cmul(rs[(int64_t)i * k + t], yi));
    __syncthreads();
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
    reduce_partials(g.P, g.ldp, 2, g.hn2);
    if (threadIdx.x == 0) {
      g.ticket[0] = 0;
      g.st->true_num2 = ld_cg(g.hn2).x;
      g.st->b_norm2 = ld_cg(g.hn2 + 1).x;
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

cudaError_t gm_arnoldi_step(const GmresDev& g, double rel_tol, int max_iter,
                            cudaGraphConditionalHandle cond, cudaStream_t s) {
  const int64_t chunk = (g.n + g.arn_blocks - 1) / g.arn_blocks;
  const size_t smem = (size_t)(ARN_SMEM_VECS * g.ldp + chunk + g.arn_vcap) * sizeof(double2);
  count_launch();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(g.arn_blocks);
  cfg.blockDim = dim3(ARN_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_arnoldi, g, rel_tol, max_iter, cond);
}

cudaError_t gm_arnoldi_setup(GmresDev& g, int device) {
  int nsm = 0;
  cudaError_t e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return e;
  g.arn_blocks = nsm < ARN_MAX_BLOCKS ? nsm : ARN_MAX_BLOCKS;
  const int64_t chunk = (g.n + g.arn_blocks - 1) / g.arn_blocks;
  int maxdyn = 0;
  e = cudaDeviceGetAttribute(&maxdyn, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (e != cudaSuccess) return e;
  const int64_t fixed = (int64_t)(ARN_SMEM_VECS * g.ldp + chunk) * (int64_t)sizeof(double2);
  g.arn_vcap = std::max<int64_t>(0, (maxdyn - 1024 - fixed) / (int64_t)sizeof(double2));
  const size_t smem = (size_t)fixed + (size_t)g.arn_vcap * sizeof(double2);
  // per-function attribute shared by every workspace: it only grows
  static std::atomic<int> attr_max{0};
  int cur = attr_max.load();
  while ((int)smem > cur && !attr_max.compare_exchange_weak(cur, (int)smem)) {
  }
  e = cudaFuncSetAttribute(k_arnoldi, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           cur > (int)smem ? cur : (int)smem);
  if (e != cudaSuccess) return e;
  // every kernel of the solve prefers the executor's shared-memory carveout:
  // no SM reconfiguration between the graph's kernels
  for (const void* f : {(const void*)k_arnoldi, (const void*)k_begin_norm, (const void*)k_begin_scale,
                        (const void*)k_backsolve, (const void*)k_combine, (const void*)k_resid,
                        (const void*)k_zero}) {
    e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                             (int)cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
  }
  {  // back substitution: R (k x k, k <= max_iter) and g in shared memory
    static std::atomic<int> bs_max{0};
    const int need = (int)((size_t)g.max_iter * (g.max_iter + 1) * sizeof(double2));
    int cur = bs_max.load();
    while (need > cur && !bs_max.compare_exchange_weak(cur, need)) {
    }
    e = cudaFuncSetAttribute(k_backsolve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             cur > need ? cur : need);
    if (e != cudaSuccess) return e;
  }
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_arnoldi, ARN_THREADS, smem);
  if (e != cudaSuccess) return e;
  return occ >= 1 ? cudaSuccess : cudaErrorInvalidConfiguration;
}

void gm_begin(const GmresDev& g, cudaGraphConditionalHandle cond, cudaStream_t s) {
  count_launch();
  k_begin_norm<<<RED_BLOCKS, RED_THREADS, 0, s>>>(g, cond);
  count_launch();
  k_begin_scale<<<grid_for(g.n), 256, 0, s>>>(g);
}

void gm_finish(const GmresDev& g, double2* x, cudaStream_t s) {
  count_launch();
  k_backsolve<<<1, RED_THREADS, (size_t)g.max_iter * (g.max_iter + 1) * sizeof(double2), s>>>(g);
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
