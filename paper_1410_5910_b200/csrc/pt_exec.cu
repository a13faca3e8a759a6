// Persistent dataflow executor for interface-operator programs.
//
// One launch runs a whole program (an A-apply, a preconditioner apply of
// n_it Gauss-Seidel sweeps, or a fused A -> M GMRES iteration).  CTAs pull
// task indices from a global queue in priority order (topological: every
// dependency of task q sits at an index < q), wait on the counters of the
// producer groups they read, compute, and bump their own group's counter.
// The launch is cooperative, so every CTA is resident and a CTA waiting on a
// counter always has a running producer: no deadlock, no grid barrier, and
// the sequential sweep chain overlaps the independent A-apply / R-term work.
//
// Kernel data is streamed with ld.global.nc.L1::no_allocate (16-byte complex
// loads, coalesced along rows); vectors written during the launch are read
// through L2 (ld.cg).  Each output element is produced by one CTA in a fixed
// order, so repeated applies are bitwise identical (no float atomics).
#include "pt_device.cuh"

namespace pt {

namespace {

__device__ __forceinline__ const double2* vptr(const ExecArgs& a, const VecRef& r) {
  return a.slot[r.slot] + r.off;
}
__device__ __forceinline__ double2* vptr_w(const ExecArgs& a, const VecRef& r) {
  return a.slot[r.slot] + r.off;
}

// rows of one output block from dense kernel terms: warp per row pair,
// lanes across columns, source (x_a [+ x_b]) staged once per term in smem.
__device__ void run_y_dense(const ExecArgs& a, const DevTask& t, double2* s) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = a.m;
  const int row0 = t.r0 + warp * DENSE_RPW;
  bool valid[DENSE_RPW];
  double2 acc[DENSE_RPW];
#pragma unroll
  for (int k = 0; k < DENSE_RPW; ++k) {
    valid[k] = row0 + k < t.r1;
    acc[k] = make_double2(0.0, 0.0);
    if (t.has_init && valid[k]) acc[k] = ld_cg(vptr(a, t.init) + row0 + k);
  }
  for (int it = 0; it < t.nterm; ++it) {
    const DevTerm tm = a.terms[t.term0 + it];
    __syncthreads();
    const double2* s0 = vptr(a, tm.src[0]);
    if (tm.nsrc > 1) {
      const double2* s1 = vptr(a, tm.src[1]);
      for (int c = threadIdx.x; c < m; c += EXEC_THREADS) s[c] = cadd(ld_cg(s0 + c), ld_cg(s1 + c));
    } else {
      for (int c = threadIdx.x; c < m; c += EXEC_THREADS) s[c] = ld_cg(s0 + c);
    }
    __syncthreads();
    if (!valid[0]) continue;
    const double2* K = a.dense + (size_t)tm.kernel * m * m + (size_t)row0 * m;
    double2 d[DENSE_RPW];
#pragma unroll
    for (int k = 0; k < DENSE_RPW; ++k) d[k] = make_double2(0.0, 0.0);
    constexpr int U = 4;
    for (int c0 = lane; c0 < m; c0 += 32 * U) {
      double2 kv[DENSE_RPW][U], sv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + 32 * u;
        const bool in = c < m;
        sv[u] = in ? s[c] : make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < DENSE_RPW; ++k)
          kv[k][u] = (in && valid[k]) ? ld_stream(K + (size_t)k * m + c) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < DENSE_RPW; ++k) d[k] = cfma(kv[k][u], sv[u], d[k]);
    }
    const double2 sc = make_double2(tm.scale_re, tm.scale_im);
#pragma unroll
    for (int k = 0; k < DENSE_RPW; ++k) {
      const double2 r = warp_sum(d[k]);
      acc[k] = cfma(sc, r, acc[k]);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < DENSE_RPW; ++k) {
      if (!valid[k]) continue;
      const int row = row0 + k;
      double2 v = acc[k];
      for (int e = 0; e < t.neye; ++e) {
        const DevEye ey = a.eyes[t.eye0 + e];
        v = cfma(make_double2(ey.re, ey.im), ld_cg(vptr(a, ey.src) + row), v);
      }
      if (t.has_rhs) {
        const double2 r = ld_cg(vptr(a, t.rhs) + row);
        v.x = fma(t.rhs_coef, r.x, v.x);
        v.y = fma(t.rhs_coef, r.y, v.y);
      }
      st_cg(vptr_w(a, t.out) + row, v);
    }
  }
}

// t = scale * Vt (x_a [+ x_b]) for a slot range of one PLR term.  The
// source (sum) is staged once in smem; warp per Vt row, lanes across columns.
// The term's scale is folded into t so the Y phase is a plain U t sum.
__device__ void run_t_plr(const ExecArgs& a, const DevTask& t, double2* s) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = a.m;
  const DevTerm tm = a.terms[t.term0];
  const DevKernelPLR kp = a.kplr[tm.kernel];
  double2* T = a.slot[SLOT_T] + tm.t_base;
  const double2* s0 = vptr(a, tm.src[0]);
  if (tm.nsrc > 1) {
    const double2* s1 = vptr(a, tm.src[1]);
    for (int c = threadIdx.x; c < m; c += EXEC_THREADS) s[c] = cadd(ld_cg(s0 + c), ld_cg(s1 + c));
  } else {
    for (int c = threadIdx.x; c < m; c += EXEC_THREADS) s[c] = ld_cg(s0 + c);
  }
  __syncthreads();
  const double2 sc = make_double2(tm.scale_re, tm.scale_im);
  for (int q = t.r0 + warp; q < t.r1; q += EXEC_WARPS) {
    const DevSlot sl = a.slots[kp.slot0 + q];
    const double2* V = a.fac + sl.v_off;
    const double2* x = s + sl.col_off;
    double2 d = make_double2(0.0, 0.0);
    constexpr int U = 4;
    for (int c0 = lane; c0 < sl.cols; c0 += 32 * U) {
      double2 vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + 32 * u;
        vv[u] = c < sl.cols ? ld_stream(V + c) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + 32 * u;
        if (c < sl.cols) d = cfma(vv[u], x[c], d);
      }
    }
    d = warp_sum(d);
    if (lane == 0) st_cg(T + q, cmul(sc, d));
  }
}

// One PLR_TILE-row tile of an output block: y_r = init + sum over terms and
// over the leaves meeting the tile of U_leaf[r, :] t_leaf (+ eyes, rhs).
// Lane = row (U is column-major: a warp reads 32 consecutive rows of one
// rank column, 512 contiguous bytes); the tile's (leaf, column) pairs are
// dealt round-robin to the 8 warps and the 8 partial sums per row are added
// in warp order.
__device__ void run_y_plr(const ExecArgs& a, const DevTask& t, double2* s) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = t.r0 + lane;
  const int tile = t.r0 / PLR_TILE;
  double2 acc = make_double2(0.0, 0.0);
  for (int it = 0; it < t.nterm; ++it) {
    const DevTerm tm = a.terms[t.term0 + it];
    const DevKernelPLR kp = a.kplr[tm.kernel];
    const double2* T = a.slot[SLOT_T] + tm.t_base;
    const int l0 = a.tile_ptr[kp.tile0 + tile], l1 = a.tile_ptr[kp.tile0 + tile + 1];
    int flat = 0;  // running index of (leaf, column) pairs within this term
    for (int l = l0; l < l1; ++l) {
      const DevLeaf lf = a.leaves[a.tile_leaves[l]];
      const int lr = row - lf.row_off;
      const bool in = lr >= 0 && lr < lf.rows;
      const double2* U = a.fac + lf.u_off + lr;
      const double2* tt = T + lf.slot0;
      int c = ((warp - flat) % EXEC_WARPS + EXEC_WARPS) % EXEC_WARPS;
      flat += lf.rank;
      for (; c + 3 * EXEC_WARPS < lf.rank; c += 4 * EXEC_WARPS) {
        double2 uv[4], tv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uv[u] = in ? ld_stream(U + (size_t)(c + u * EXEC_WARPS) * lf.rows) : make_double2(0.0, 0.0);
          tv[u] = ld_cg(tt + c + u * EXEC_WARPS);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc = cfma(uv[u], tv[u], acc);
      }
      for (; c < lf.rank; c += EXEC_WARPS) {
        const double2 uv = in ? ld_stream(U + (size_t)c * lf.rows) : make_double2(0.0, 0.0);
        acc = cfma(uv, ld_cg(tt + c), acc);
      }
    }
  }
  s[warp * 32 + lane] = acc;
  __syncthreads();
  if (warp != 0 || row >= t.r1) return;
  double2 v = make_double2(0.0, 0.0);
  if (t.has_init) v = ld_cg(vptr(a, t.init) + row);
#pragma unroll
  for (int w = 0; w < EXEC_WARPS; ++w) v = cadd(v, s[w * 32 + lane]);
  for (int e = 0; e < t.neye; ++e) {
    const DevEye ey = a.eyes[t.eye0 + e];
    v = cfma(make_double2(ey.re, ey.im), ld_cg(vptr(a, ey.src) + row), v);
  }
  if (t.has_rhs) {
    const double2 r = ld_cg(vptr(a, t.rhs) + row);
    v.x = fma(t.rhs_coef, r.x, v.x);
    v.y = fma(t.rhs_coef, r.y, v.y);
  }
  st_cg(vptr_w(a, t.out) + row, v);
}

}  // namespace

__global__ void __launch_bounds__(EXEC_THREADS) pt_exec_kernel(ExecArgs a) {
  extern __shared__ double2 smem[];
  __shared__ int s_task;
  if (a.stop) {
    if (threadIdx.x == 0) s_task = *((volatile const int*)a.stop);
    __syncthreads();
    if (s_task) return;
    __syncthreads();
  }
  if (a.iter) {
    const int64_t j = *((volatile const int*)a.iter);
    a.slot[SLOT_IN] = a.vbase + j * a.vstride;
    a.slot[SLOT_OUT] = a.vbase + (j + 1) * a.vstride;
  }
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(a.head, 1);
    __syncthreads();
    const int q = s_task;
    if (q >= a.n_tasks) return;
    const DevTask t = a.tasks[q];
    if (threadIdx.x == 0) {
      for (int w = 0; w < t.nwait; ++w) {
        const DevWait dw = a.waits[t.wait0 + w];
        while (ld_acquire(a.ctr + dw.ctr) < dw.val) __nanosleep(32);
      }
    }
    __syncthreads();
    if (t.type == TASK_Y_DENSE)
      run_y_dense(a, t, smem);
    else if (t.type == TASK_T_PLR)
      run_t_plr(a, t, smem);
    else
      run_y_plr(a, t, smem);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(a.ctr + t.signal, 1);
    }
  }
}

}  // namespace pt
