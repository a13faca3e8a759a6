// Batched (multi-RHS) executor and GMRES kernels.  See pt_batch.cuh.
//
// The executor runs the same task DAG the host plan builder makes for the
// single-source executor (pt_plan.cpp: queue order, producer-group counters,
// row-chunk dependencies), built with BT_ROWS-row dense tasks.  A task
// computes BT_ROWS output rows for all BW sources:
//   out = sum_terms K[rows, :] . (scale (X_a [+ X_b])) + init + sum eye X + c rhs
// Per task the CTA streams K in BT_KC-column chunks with cp.async (16-byte,
// zero-filled at the ragged edges) and stages scale (X_a + X_b) for the
// chunk's rows through registers (L2 loads: X is produced inside the launch),
// double-buffered so the next chunk's loads overlap the current chunk's
// DMMA work.  Complex products are four real m8n8k4 DMMAs per fragment.
// Each output element is owned by one CTA and summed in a fixed order: the
// batched applies are bitwise repeatable.
//
// GMRES (solver.py:231-295, per source): CGS2 + Givens with the flags of
// :265-289, every source in lockstep with its own status; a stopped source
// is frozen (its next basis column is zeroed and its report no longer
// changes), so each source's iterations equal its own single solve's.
#include <algorithm>
#include <cmath>

#include "pt_batch.cuh"

namespace pt {

extern void count_launch();

namespace {

constexpr int AS_LD = BT_KC + 4;  // A rows 4 apart mod 8 (16-byte units): conflict-free fragments
// X chunk rows: COLS + 2 complex (2 apart mod 8 in 16-byte units: conflict-free B fragments)
template <int COLS>
constexpr int xs_ld() { return COLS + 2; }
template <int ROWS, int COLS>
constexpr size_t bexec_smem() {
  return (size_t)(2 * ROWS * AS_LD + 2 * BT_KC * xs_ld<COLS>()) * sizeof(double2);
}
static_assert(BW == 64 && BT_THREADS == 256, "warp tiling assumes 8 warps over 64 sources");

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// 16-byte async copy; bytes = 0 zero-fills the destination
__device__ __forceinline__ void cp16z(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// d += a * b on an 8x8x4 FP64 tensor-core tile (A row, B col fragments)
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// A task covers ROWS output rows and COLS of the 64 sources (columns
// [c0, c0 + COLS), c0 = the task's c0 field).  ROWS x COLS = 16 x 64: 8 warps =
// 2 row groups x 4 column groups of 16 sources (two n-tiles each); 8 x 64:
// 1 x 8 groups of 8 sources; 16 x 32: 2 x 4 groups of 8 sources.
template <int ROWS, int COLS>
__global__ void __launch_bounds__(BT_THREADS, BT_CTAS_PER_SM) pt_bexec_kernel(BExecArgs a) {
  constexpr int RG = ROWS / 8;           // row groups of 8
  constexpr int CG = 8 / RG;             // column groups
  constexpr int NT = COLS / CG / 8;      // n-tiles (8 sources) per warp
  constexpr int XU = COLS / 16;          // X values per thread per chunk (16 threads per row)
  constexpr int XS_LD = xs_ld<COLS>();
  constexpr int XS_ELEMS = BT_KC * XS_LD;
  static_assert(NT >= 1 && BT_KC * COLS == XU * BT_THREADS, "tiling");
  constexpr int AS_ELEMS = ROWS * AS_LD;
  extern __shared__ __align__(16) double2 bsm[];
  double2* As = bsm;                 // [2][ROWS][AS_LD]  kernel rows of the chunk
  double2* Xs = bsm + 2 * AS_ELEMS;  // [2][BT_KC][XS_LD] scaled sources of the chunk
  __shared__ double2* s_vec[N_SLOTS];
  __shared__ DevTask s_task;
  __shared__ DevTerm s_terms[BT_TERMS];
  __shared__ DevEye s_eyes[BT_EYES];
  __shared__ int s_q, s_stop;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_stop = a.stop ? *((volatile const int*)a.stop) : 0;
  if (tid < N_SLOTS) {
    double2* p = a.slot[tid];
    if (a.iter && (tid == SLOT_IN || tid == SLOT_OUT)) {
      const int64_t j = *((volatile const int*)a.iter) + (tid == SLOT_OUT ? 1 : 0);
      p = a.vbase + j * a.vstride;
    }
    s_vec[tid] = p;
  }
  __syncthreads();
  if (s_stop) return;
  const int m = a.m;
  const int kchunks = (m + BT_KC - 1) / BT_KC;
  const int wr = (wid % RG) * 8;         // the warp's 8 output rows
  const int wc = (wid / RG) * (NT * 8);  // the warp's first output column
  const int kr = tid >> 4, xc = tid & 15;  // X staging: chunk row, columns xc + 16u
  const int ar = tid / BT_KC, ak = tid % BT_KC;  // A staging: one 16-byte copy (ar < ROWS)
  for (;;) {
    if (tid == 0) s_q = atomicAdd(a.head, 1);
    __syncthreads();
    const int q = s_q;
    if (q >= a.n_tasks) return;
    if (tid < (int)(sizeof(DevTask) / 4))
      reinterpret_cast<int*>(&s_task)[tid] = __ldg(reinterpret_cast<const int*>(a.tasks + q) + tid);
    __syncthreads();
    const int nterm = s_task.nterm, neye = s_task.neye;
    if (tid < nterm) s_terms[tid] = a.terms[s_task.term0 + tid];
    if (tid >= 32 && tid < 32 + neye) s_eyes[tid - 32] = a.eyes[s_task.eye0 + tid - 32];
    if (wid == 2) {  // dependencies: the lanes poll the task's counters
      const DevWait* w = a.waits + s_task.wait0;
      const int nw = s_task.nwait;
      bool ok;
      do {
        ok = true;
        for (int i = lane; i < nw; i += 32)
          if (ld_acquire(a.ctr + w[i].ctr) < w[i].val) ok = false;
        ok = __all_sync(0xffffffffu, ok);
        if (!ok) __nanosleep(32);
      } while (!ok);
    }
    __syncthreads();
    const int r0 = s_task.r0, nrows = s_task.r1 - s_task.r0;
    const int cb = COLS == BW ? 0 : s_task.c0;  // the task's first source column
    const int nch = nterm * kchunks;

    auto load_A = [&](int c, int buf) {
      if (ar < ROWS) {
        const int term = c / kchunks, kc = (c - term * kchunks) * BT_KC;
        const double2* K = a.dense + ((size_t)s_terms[term].kernel * m + r0) * (size_t)m;
        const bool ok = ar < nrows && kc + ak < m;
        cp16z(As + buf * AS_ELEMS + ar * AS_LD + ak, ok ? K + (size_t)ar * m + kc + ak : K,
              ok ? 16 : 0);
      }
      cp_commit();
    };
    double2 xa[XU], xb[XU];
    auto load_X = [&](int c) {
      const int term = c / kchunks, kc = (c - term * kchunks) * BT_KC;
      const DevTerm& tm = s_terms[term];
      const int64_t row = kc + kr;
#pragma unroll
      for (int u = 0; u < XU; ++u) xa[u] = xb[u] = make_double2(0.0, 0.0);
      if (row < m) {
        const double2* p0 = s_vec[tm.src[0].slot] + (tm.src[0].off + row) * BW + cb + xc;
#pragma unroll
        for (int u = 0; u < XU; ++u) xa[u] = ld_cg(p0 + 16 * u);
        if (tm.nsrc > 1) {
          const double2* p1 = s_vec[tm.src[1].slot] + (tm.src[1].off + row) * BW + cb + xc;
#pragma unroll
          for (int u = 0; u < XU; ++u) xb[u] = ld_cg(p1 + 16 * u);
        }
      }
    };
    auto store_X = [&](int c, int buf) {
      const DevTerm& tm = s_terms[c / kchunks];
      const double2 sc = make_double2(tm.scale_re, tm.scale_im);
      double2* d = Xs + buf * XS_ELEMS + kr * XS_LD + xc;
#pragma unroll
      for (int u = 0; u < XU; ++u) d[16 * u] = cmul(sc, cadd(xa[u], xb[u]));
    };
    double acc[NT][2][2];  // [n-tile][re, im][pair]
#pragma unroll
    for (int u = 0; u < NT; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v) acc[u][v][0] = acc[u][v][1] = 0.0;
    auto compute = [&](int buf) {
      const double2* Ab = As + buf * AS_ELEMS + (wr + (lane >> 2)) * AS_LD + (lane & 3);
      const double2* Xb = Xs + buf * XS_ELEMS + (lane & 3) * XS_LD + wc + (lane >> 2);
#pragma unroll
      for (int ks = 0; ks < BT_KC / 4; ++ks) {
        const double2 av = Ab[ks * 4];
        const double nai = -av.y;
#pragma unroll
        for (int u = 0; u < NT; ++u) {
          const double2 bv = Xb[ks * 4 * XS_LD + u * 8];
          dmma(acc[u][0], av.x, bv.x);
          dmma(acc[u][0], nai, bv.y);
          dmma(acc[u][1], av.x, bv.y);
          dmma(acc[u][1], av.y, bv.x);
        }
      }
    };
    if (nch > 0) {
      load_A(0, 0);
      load_X(0);
      store_X(0, 0);
    }
    for (int c = 0; c < nch; ++c) {
      cp_wait_all();
      __syncthreads();  // chunk c staged; every warp done with chunk c - 1
      const bool more = c + 1 < nch;
      if (more) {
        load_A(c + 1, (c + 1) & 1);
        load_X(c + 1);
      }
      compute(c & 1);
      if (more) store_X(c + 1, (c + 1) & 1);
    }
    // epilogue: rows wr + lane/4, columns wc + 8u + 2(lane%4) + e
    const int orow = wr + (lane >> 2);
    if (orow < nrows) {
      const int64_t rb = (int64_t)(r0 + orow) * BW + cb;
      double2* outp = s_vec[s_task.out.slot] + s_task.out.off * BW + rb;
      const double2* initp = s_task.has_init ? s_vec[s_task.init.slot] + s_task.init.off * BW + rb : nullptr;
      const double2* rhsp = s_task.has_rhs ? s_vec[s_task.rhs.slot] + s_task.rhs.off * BW + rb : nullptr;
      const double rc = s_task.rhs_coef;
#pragma unroll
      for (int u = 0; u < NT; ++u) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = wc + 8 * u + 2 * (lane & 3) + e;
          double2 v = make_double2(0.0, 0.0);
          if (initp) v = ld_cg(initp + col);
          for (int i = 0; i < neye; ++i) {
            const DevEye& ey = s_eyes[i];
            v = cfma(make_double2(ey.re, ey.im),
                     ld_cg(s_vec[ey.src.slot] + ey.src.off * BW + rb + col), v);
          }
          if (rhsp) {
            const double2 r = ld_cg(rhsp + col);
            v.x = fma(rc, r.x, v.x);
            v.y = fma(rc, r.y, v.y);
          }
          v.x += acc[u][0][e];
          v.y += acc[u][1][e];
          st_cg(outp + col, v);
        }
      }
    }
    __syncthreads();
    if (tid == 0 && s_task.signal >= 0) {
      __threadfence();
      asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.ctr + s_task.signal) : "memory");
    }
  }
}

// ---- batched GMRES ------------------------------------------------------------
// Row-parallel kernels: BRED_BLOCKS blocks of 256 threads = 4 row groups x
// BW sources (thread = (row group, source)); per-block partials are reduced
// in a fixed order, so every result is bitwise repeatable.

constexpr int BG_THREADS = 256;
constexpr int BG_RG = BG_THREADS / BW;  // row groups per block
constexpr int BG_CH = 8;                // basis columns per dots pass
constexpr int BR_THREADS = 512;         // reductions: 8 groups x BW sources
constexpr int BR_G = BR_THREADS / BW;

__device__ __forceinline__ void rows_of_block(int64_t n, int64_t& lo, int64_t& hi) {
  const int64_t chunk = (n + BRED_BLOCKS - 1) / BRED_BLOCKS;
  lo = (int64_t)blockIdx.x * chunk;
  hi = lo + chunk < n ? lo + chunk : n;
  if (lo > n) lo = n;
}
__device__ __forceinline__ int64_t pidx(const BGmresDev& g, int blk, int i, int s) {
  return ((int64_t)blk * (g.max_iter + 1) + i) * BW + s;
}
__device__ __forceinline__ double2* col(const BGmresDev& g, int j) {
  return g.V + (int64_t)j * g.n * BW;
}
__device__ __forceinline__ bool all_stopped(const BGmresDev& g) {
  return *((volatile const int*)(g.ctl + 1)) != 0;
}

// P[blk, i, s] = sum over the block's rows of conj(V_i[r, s]) w[r, s], i <= j;
// pass 1 also flags non-finite values of live sources
__global__ void __launch_bounds__(BG_THREADS) k_bdots(BGmresDev g, int pass) {
  if (all_stopped(g)) return;
  __shared__ double2 red[BG_RG][BG_CH][BW];
  const int s = threadIdx.x % BW, rg = threadIdx.x / BW;
  const int j = g.ctl[0], nc = j + 1;
  const double2* w = col(g, j + 1);
  int64_t lo, hi;
  rows_of_block(g.n, lo, hi);
  if (pass == 1 && !g.st[s].stop) {
    bool bad = false;
    for (int64_t r = lo + rg; r < hi; r += BG_RG) {
      const double2 v = ld_cg(w + r * BW + s);
      bad |= !(isfinite(v.x) && isfinite(v.y));
    }
    if (bad) atomicOr(&g.st[s].nonfinite, 1);
  }
  for (int c0 = 0; c0 < nc; c0 += BG_CH) {
    const int cnt = nc - c0 < BG_CH ? nc - c0 : BG_CH;
    double2 acc[BG_CH];
#pragma unroll
    for (int u = 0; u < BG_CH; ++u) acc[u] = make_double2(0.0, 0.0);
    for (int64_t r = lo + rg; r < hi; r += BG_RG) {
      const double2 wv = ld_cg(w + r * BW + s);
#pragma unroll
      for (int u = 0; u < BG_CH; ++u)
        if (u < cnt) acc[u] = cfma_conj(ld_cg(col(g, c0 + u) + r * BW + s), wv, acc[u]);
    }
#pragma unroll
    for (int u = 0; u < BG_CH; ++u) red[rg][u][s] = acc[u];
    __syncthreads();
    if (rg == 0)
      for (int u = 0; u < cnt; ++u) {
        double2 t = red[0][u][s];
        for (int k = 1; k < BG_RG; ++k) t = cadd(t, red[k][u][s]);
        st_cg(g.P + pidx(g, blockIdx.x, c0 + u, s), t);
      }
    __syncthreads();
  }
}

// out[i, s] = sum over blocks (fixed order) of P[blk, i, s]; block i, i <= ncols - 1
__global__ void __launch_bounds__(BR_THREADS) k_bred(BGmresDev g, double2* out, int fixed_cols) {
  if (all_stopped(g)) return;
  const int nc = fixed_cols > 0 ? fixed_cols : g.ctl[0] + 1;
  const int i = blockIdx.x;
  if (i >= nc) return;
  __shared__ double2 red[BR_G][BW];
  const int s = threadIdx.x % BW, gq = threadIdx.x / BW;
  double2 t = make_double2(0.0, 0.0);
  for (int b = gq; b < BRED_BLOCKS; b += BR_G) t = cadd(t, ld_cg(g.P + pidx(g, b, i, s)));
  red[gq][s] = t;
  __syncthreads();
  if (gq == 0) {
    double2 u = red[0][s];
    for (int k = 1; k < BR_G; ++k) u = cadd(u, red[k][s]);
    st_cg(out + (int64_t)i * BW + s, u);
  }
}

// w -= sum_i V_i h[i] (i <= j); with norm: P[blk, 0, s].x = ||w[:, s]||^2 partial
__global__ void __launch_bounds__(BG_THREADS) k_bupd(BGmresDev g, const double2* h, int norm) {
  if (all_stopped(g)) return;
  __shared__ double red[BG_RG][BW];
  const int s = threadIdx.x % BW, rg = threadIdx.x / BW;
  const int j = g.ctl[0], nc = j + 1;
  double2* w = col(g, j + 1);
  int64_t lo, hi;
  rows_of_block(g.n, lo, hi);
  double nn = 0.0;
  for (int64_t r = lo + rg; r < hi; r += BG_RG) {
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < nc; ++i) acc = cfma(ld_cg(col(g, i) + r * BW + s), __ldg(h + (int64_t)i * BW + s), acc);
    const double2 v = csub(ld_cg(w + r * BW + s), acc);
    st_cg(w + r * BW + s, v);
    nn = fma(v.x, v.x, nn);
    nn = fma(v.y, v.y, nn);
  }
  if (!norm) return;
  red[rg][s] = nn;
  __syncthreads();
  if (rg == 0) {
    double t = red[0][s];
    for (int k = 1; k < BG_RG; ++k) t += red[k][s];
    st_cg(g.P + pidx(g, blockIdx.x, 0, s), make_double2(t, 0.0));
  }
}

// P[blk, 0, s] = (||v||^2, 0) partials of one batched vector
__global__ void __launch_bounds__(BG_THREADS) k_bnorm(BGmresDev g, const double2* v) {
  __shared__ double red[BG_RG][BW];
  const int s = threadIdx.x % BW, rg = threadIdx.x / BW;
  int64_t lo, hi;
  rows_of_block(g.n, lo, hi);
  double nn = 0.0;
  for (int64_t r = lo + rg; r < hi; r += BG_RG) {
    const double2 x = ld_cg(v + r * BW + s);
    nn = fma(x.x, x.x, nn);
    nn = fma(x.y, x.y, nn);
  }
  red[rg][s] = nn;
  __syncthreads();
  if (rg == 0) {
    double t = red[0][s];
    for (int k = 1; k < BG_RG; ++k) t += red[k][s];
    st_cg(g.P + pidx(g, blockIdx.x, 0, s), make_double2(t, 0.0));
  }
}

// fixed-order sum of the P[blk, 0, s] partials into sm[s] (one block of BR_THREADS)
__device__ void reduce_norm_partials(const BGmresDev& g, double2* sm, double2 (*red)[BW]) {
  const int s = threadIdx.x % BW, gq = threadIdx.x / BW;
  double2 t = make_double2(0.0, 0.0);
  for (int b = gq; b < BRED_BLOCKS; b += BR_G) t = cadd(t, ld_cg(g.P + pidx(g, b, 0, s)));
  red[gq][s] = t;
  __syncthreads();
  if (gq == 0) {
    double2 u = red[0][s];
    for (int k = 1; k < BR_G; ++k) u = cadd(u, red[k][s]);
    sm[s] = u;
  }
  __syncthreads();
}

// beta_s = ||M^-1 b_s||, statuses, g = beta e1 (solver.py:236-246 per source)
__global__ void __launch_bounds__(BR_THREADS) k_bbegin(BGmresDev g, cudaGraphConditionalHandle cond) {
  __shared__ double2 red[BR_G][BW];
  __shared__ double2 nn[BW];
  reduce_norm_partials(g, nn, red);
  const int s = threadIdx.x;
  if (s < BW) {
    DevStatus& st = g.st[s];
    const double beta = sqrt(nn[s].x);
    st.iterations = 0;
    st.flag = 0;
    st.nonfinite = 0;
    st.breakdown = 0;
    st.rel = 1.0;
    st.beta = beta;
    st.hn = beta;
    st.true_num2 = 0.0;
    st.b_norm2 = 0.0;
    // beta == 0 (or a padding column): x = 0, converged (solver.py:239-242)
    const bool zero = beta == 0.0 || s >= g.nrhs;
    st.converged = zero ? 1 : 0;
    st.stop = zero ? 1 : 0;
    st.inv_hn = zero ? 0.0 : 1.0 / beta;
    g.inv[s] = st.inv_hn;
    double2* gs = g.g + (int64_t)s * (g.max_iter + 1);
    for (int i = 0; i <= g.max_iter; ++i) gs[i] = make_double2(0.0, 0.0);
    gs[0] = make_double2(beta, 0.0);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int all = 1;
    for (int k = 0; k < BW; ++k) all &= g.st[k].stop;
    g.ctl[0] = 0;
    g.ctl[1] = all;
    g.ctl[2] = 0;
    __threadfence();
    if (cond) cudaGraphSetConditional(cond, all ? 0u : 1u);
  }
}

// Arnoldi column j of every live source: h = h1 + h2, ||w||, Givens, flags
// (the single-source givens_update of pt_gmres.cu, per source)
__global__ void __launch_bounds__(BR_THREADS)
k_bgivens(BGmresDev g, double rel_tol, int max_iter, cudaGraphConditionalHandle cond) {
  if (all_stopped(g)) return;
  __shared__ double2 red[BR_G][BW];
  __shared__ double2 nn[BW];
  reduce_norm_partials(g, nn, red);
  const int j = g.ctl[0];
  const int s = threadIdx.x;
  if (s < BW) {
    DevStatus& st = g.st[s];
    double inv = 0.0;
    if (!st.stop && st.nonfinite) {
      st.stop = 1;
      st.converged = 0;
    } else if (!st.stop) {
      const int ldr = g.max_iter + 1;
      double2* Rj = g.R + (int64_t)s * ldr * g.max_iter + (int64_t)j * ldr;
      double* cs = g.cs + (int64_t)s * g.max_iter;
      double2* sn = g.sn + (int64_t)s * g.max_iter;
      double2* gs = g.g + (int64_t)s * ldr;
      double* hist = g.hist + (int64_t)s * g.max_iter;
      const double hn = sqrt(nn[s].x);
      // previous rotations applied down the new column, carried in registers
      double2 a = cadd(ld_cg(g.h1 + s), ld_cg(g.h2 + s));
      for (int i = 0; i < j; ++i) {
        const double2 b = cadd(ld_cg(g.h1 + (int64_t)(i + 1) * BW + s), ld_cg(g.h2 + (int64_t)(i + 1) * BW + s));
        const double c = cs[i];
        const double2 sv = sn[i];
        Rj[i] = cadd(make_double2(c * a.x, c * a.y), cmul(sv, b));
        a = cadd(cmul(make_double2(-sv.x, sv.y), a), make_double2(c * b.x, c * b.y));
      }
      const double aa = sqrt(a.x * a.x + a.y * a.y);
      double c;
      double2 sv, rr;
      if (aa == 0.0 && hn == 0.0) {
        c = 1.0;
        sv = make_double2(0.0, 0.0);
        rr = make_double2(0.0, 0.0);
      } else if (aa == 0.0) {
        c = 0.0;
        sv = make_double2(1.0, 0.0);
        rr = make_double2(hn, 0.0);
      } else {
        const double r = hypot(aa, hn);
        const double2 ph = make_double2(a.x / aa, a.y / aa);
        c = aa / r;
        sv = make_double2(ph.x * hn / r, ph.y * hn / r);
        rr = make_double2(ph.x * r, ph.y * r);
      }
      cs[j] = c;
      sn[j] = sv;
      Rj[j] = rr;
      Rj[j + 1] = make_double2(0.0, 0.0);
      const double2 gj = gs[j];
      gs[j] = make_double2(c * gj.x, c * gj.y);
      gs[j + 1] = cmul(make_double2(-sv.x, sv.y), gj);
      const double beta = st.beta;
      const double2 gn = gs[j + 1];
      const double rel = sqrt(gn.x * gn.x + gn.y * gn.y) / beta;
      hist[j] = rel;
      const int k = j + 1;
      st.iterations = k;
      st.rel = rel;
      st.hn = hn;
      const bool breakdown = hn <= BREAKDOWN_REL * beta;  // solver.py:265
      st.breakdown = breakdown ? 1 : 0;
      st.inv_hn = breakdown ? 0.0 : 1.0 / hn;
      inv = st.inv_hn;
      if (breakdown) {
        st.converged = 1;
        st.flag = 1;
        st.stop = 1;
      } else if (rel <= rel_tol) {  // solver.py:279
        st.converged = 1;
        st.flag = 0;
        st.stop = 1;
      } else if (k > STAG_WINDOW && hist[k - 1 - STAG_WINDOW] > 0.0 &&  // solver.py:282-287
                 1.0 - rel / hist[k - 1 - STAG_WINDOW] < STAG_IMPROVEMENT) {
        st.flag = 2;
        st.stop = 1;
      } else if (k >= max_iter) {  // for/else, solver.py:288-289
        st.flag = 3;
        st.stop = 1;
      }
      // a source that stops here keeps a zero next column (frozen)
      if (st.stop) inv = 0.0;
    }
    g.inv[s] = inv;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int all = 1, bad = 0;
    for (int k = 0; k < BW; ++k) {
      all &= g.st[k].stop;
      bad |= g.st[k].nonfinite;
    }
    g.ctl[0] = j + 1;
    g.ctl[1] = all;
    g.ctl[2] = bad;
    __threadfence();
    if (cond) cudaGraphSetConditional(cond, all ? 0u : 1u);
  }
}

// V_j[:, s] *= inv[s], j = ctl[0] (the column just produced)
__global__ void k_bscale(BGmresDev g) {
  const int j = g.ctl[0];
  double2* v = col(g, j);
  const int64_t total = g.n * BW;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double sc = __ldg(g.inv + (e % BW));
    double2 x = make_double2(0.0, 0.0);  // exact zero for a stopped source (even a non-finite one)
    if (sc != 0.0) {
      x = ld_cg(v + e);
      x.x *= sc;
      x.y *= sc;
    }
    st_cg(v + e, x);
  }
}

// R_s y_s = g_s[0:k_s] (block s; the single-source k_backsolve per source)
__global__ void __launch_bounds__(RED_THREADS) k_bbacksolve(BGmresDev g) {
  extern __shared__ double2 rs[];
  const int s = blockIdx.x;
  const int k = g.st[s].iterations;
  const int ldr = g.max_iter + 1;
  const double2* R = g.R + (int64_t)s * ldr * g.max_iter;
  double2* y = g.y + (int64_t)s * g.max_iter;
  double2* gs = rs + (int64_t)k * k;
  for (int i = threadIdx.x; i < k * k; i += blockDim.x) rs[i] = R[(int64_t)(i / k) * ldr + (i % k)];
  for (int i = threadIdx.x; i < k; i += blockDim.x) gs[i] = g.g[(int64_t)s * ldr + i];
  for (int i = k + threadIdx.x; i < g.max_iter; i += blockDim.x) y[i] = make_double2(0.0, 0.0);
  __syncthreads();
  for (int i = k - 1; i >= 0; --i) {
    const double2 d = rs[(int64_t)i * k + i];
    const double dd = d.x * d.x + d.y * d.y;
    const double2 acc = gs[i];
    const double2 yi = dd == 0.0 ? make_double2(0.0, 0.0)
                                 : make_double2((acc.x * d.x + acc.y * d.y) / dd,
                                                (acc.y * d.x - acc.x * d.y) / dd);
    __syncthreads();
    if (threadIdx.x == 0) y[i] = yi;
    for (int t = threadIdx.x; t < i; t += blockDim.x) gs[t] = csub(gs[t], cmul(rs[(int64_t)i * k + t], yi));
    __syncthreads();
  }
}

// x[:, s] = V[:, :k_s] y_s
__global__ void k_bcombine(BGmresDev g, double2* x) {
  const int64_t total = g.n * BW;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(e % BW);
    const int k = g.st[s].iterations;
    const double2* y = g.y + (int64_t)s * g.max_iter;
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < k; ++i) acc = cfma(ld_cg(col(g, i) + e), __ldg(y + i), acc);
    st_cg(x + e, acc);
  }
}

// P[blk, 0, s] = (||b - Ax||^2, ||b||^2) partials
__global__ void __launch_bounds__(BG_THREADS) k_bresid(BGmresDev g, const double2* b, const double2* ax) {
  __shared__ double2 red[BG_RG][BW];
  const int s = threadIdx.x % BW, rg = threadIdx.x / BW;
  int64_t lo, hi;
  rows_of_block(g.n, lo, hi);
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t r = lo + rg; r < hi; r += BG_RG) {
    const double2 bv = ld_cg(b + r * BW + s);
    const double2 d = csub(bv, ld_cg(ax + r * BW + s));
    acc.x = fma(d.x, d.x, acc.x);
    acc.x = fma(d.y, d.y, acc.x);
    acc.y = fma(bv.x, bv.x, acc.y);
    acc.y = fma(bv.y, bv.y, acc.y);
  }
  red[rg][s] = acc;
  __syncthreads();
  if (rg == 0) {
    double2 t = red[0][s];
    for (int k = 1; k < BG_RG; ++k) t = cadd(t, red[k][s]);
    st_cg(g.P + pidx(g, blockIdx.x, 0, s), t);
  }
}

__global__ void __launch_bounds__(BR_THREADS) k_bresid_fin(BGmresDev g) {
  __shared__ double2 red[BR_G][BW];
  __shared__ double2 nn[BW];
  reduce_norm_partials(g, nn, red);
  const int s = threadIdx.x;
  if (s < BW) {
    g.st[s].true_num2 = nn[s].x;
    g.st[s].b_norm2 = nn[s].y;
  }
}

// dst[i * BW + c] = src[c * n + i] (c < ncols, zero beyond): 32 x 32 tiles
__global__ void k_bpack(const double2* src, int64_t n, int ncols, double2* dst) {
  __shared__ double2 t[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 256 threads: 8 rows per pass
  for (int r = ty; r < 32; r += 8) {  // read: column c0 + r, rows i0 + tx
    const int c = c0 + r;
    const int64_t i = i0 + tx;
    t[r][tx] = (c < ncols && i < n) ? src[(int64_t)c * n + i] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {  // write: row i0 + r, columns c0 + tx
    const int64_t i = i0 + r;
    if (i < n) dst[i * BW + c0 + tx] = t[tx][r];
  }
}
__global__ void k_bunpack(const double2* src, int64_t n, int ncols, double2* dst) {
  __shared__ double2 t[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {  // read: row i0 + r, columns c0 + tx
    const int64_t i = i0 + r;
    t[r][tx] = i < n ? src[i * BW + c0 + tx] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {  // write: column c0 + r, rows i0 + tx
    const int c = c0 + r;
    const int64_t i = i0 + tx;
    if (c < ncols && i < n) dst[(int64_t)c * n + i] = t[tx][r];
  }
}

int elem_grid(int64_t n) {
  const int64_t b = (n * BW + 255) / 256;
  return (int)std::min<int64_t>(std::max<int64_t>(b, 1), 2368);
}

}  // namespace

#define PT_BEXEC_VARIANTS(X) X(16, 64) X(8, 64) X(16, 32)

cudaError_t bexec_setup() {
  cudaError_t e = cudaSuccess;
#define PT_SETUP(R, C)                                                                      \
  if (e == cudaSuccess)                                                                     \
    e = cudaFuncSetAttribute(pt_bexec_kernel<R, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)bexec_smem<R, C>());                                      \
  if (e == cudaSuccess)                                                                     \
    e = cudaFuncSetAttribute(pt_bexec_kernel<R, C>, cudaFuncAttributePreferredSharedMemoryCarveout, \
                             (int)cudaSharedmemCarveoutMaxShared);
  PT_BEXEC_VARIANTS(PT_SETUP)
#undef PT_SETUP
  return e;
}

int bexec_grid(int device, int rows, int cols) {
  int nsm = 0, occ = 0;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  cudaError_t e = cudaErrorInvalidValue;
#define PT_OCC(R, C)                                                                          \
  if (rows == R && cols == C)                                                                 \
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pt_bexec_kernel<R, C>, BT_THREADS, \
                                                      bexec_smem<R, C>());
  PT_BEXEC_VARIANTS(PT_OCC)
#undef PT_OCC
  if (e != cudaSuccess) return 0;
  return nsm * std::max(occ, 1);
}

cudaError_t bexec_launch(const BExecArgs& a, int grid, int rows, int cols, cudaStream_t s) {
  count_launch();
#define PT_LAUNCH(R, C)                                                   \
  if (rows == R && cols == C) {                                           \
    pt_bexec_kernel<R, C><<<grid, BT_THREADS, bexec_smem<R, C>(), s>>>(a); \
    return cudaGetLastError();                                            \
  }
  PT_BEXEC_VARIANTS(PT_LAUNCH)
#undef PT_LAUNCH
  return cudaErrorInvalidValue;
}

cudaError_t bg_setup(int max_iter) {
  const int need = (int)((size_t)max_iter * (max_iter + 1) * sizeof(double2));
  return cudaFuncSetAttribute(k_bbacksolve, cudaFuncAttributeMaxDynamicSharedMemorySize, need);
}

void bg_begin(const BGmresDev& g, cudaGraphConditionalHandle cond, cudaStream_t s) {
  count_launch();
  k_bnorm<<<BRED_BLOCKS, BG_THREADS, 0, s>>>(g, g.V);
  count_launch();
  k_bbegin<<<1, BR_THREADS, 0, s>>>(g, cond);
  count_launch();
  k_bscale<<<elem_grid(g.n), 256, 0, s>>>(g);
}

void bg_step(const BGmresDev& g, double rel_tol, int max_iter, cudaGraphConditionalHandle cond,
             cudaStream_t s) {
  count_launch();
  k_bdots<<<BRED_BLOCKS, BG_THREADS, 0, s>>>(g, 1);
  count_launch();
  k_bred<<<g.max_iter + 1, BR_THREADS, 0, s>>>(g, g.h1, 0);
  count_launch();
  k_bupd<<<BRED_BLOCKS, BG_THREADS, 0, s>>>(g, g.h1, 0);
  count_launch();
  k_bdots<<<BRED_BLOCKS, BG_THREADS, 0, s>>>(g, 2);
  count_launch();
  k_bred<<<g.max_iter + 1, BR_THREADS, 0, s>>>(g, g.h2, 0);
  count_launch();
  k_bupd<<<BRED_BLOCKS, BG_THREADS, 0, s>>>(g, g.h2, 1);
  count_launch();
  k_bgivens<<<1, BR_THREADS, 0, s>>>(g, rel_tol, max_iter, cond);
  count_launch();
  k_bscale<<<elem_grid(g.n), 256, 0, s>>>(g);
}

void bg_finish(const BGmresDev& g, double2* x, cudaStream_t s) {
  count_launch();
  k_bbacksolve<<<BW, RED_THREADS, (size_t)g.max_iter * (g.max_iter + 1) * sizeof(double2), s>>>(g);
  count_launch();
  k_bcombine<<<elem_grid(g.n), 256, 0, s>>>(g, x);
}

void bg_resid(const BGmresDev& g, const double2* b, const double2* ax, cudaStream_t s) {
  count_launch();
  k_bresid<<<BRED_BLOCKS, BG_THREADS, 0, s>>>(g, b, ax);
  count_launch();
  k_bresid_fin<<<1, BR_THREADS, 0, s>>>(g);
}

void b_pack(const double2* src, int64_t n, int ncols, double2* dst, cudaStream_t s) {
  count_launch();
  k_bpack<<<dim3((unsigned)((n + 31) / 32), BW / 32), 256, 0, s>>>(src, n, ncols, dst);
}

void b_unpack(const double2* src, int64_t n, int ncols, double2* dst, cudaStream_t s) {
  count_launch();
  k_bunpack<<<dim3((unsigned)((n + 31) / 32), BW / 32), 256, 0, s>>>(src, n, ncols, dst);
}

}  // namespace pt
