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

// t = Vt (x_a [+ x_b]) for a slot range of one PLR term: warp per slot.
__device__ void run_t_plr(const ExecArgs& a, const DevTask& t) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const DevTerm tm = a.terms[t.term0];
  const DevKernelPLR kp = a.kplr[tm.kernel];
  double2* T = a.slot[SLOT_T] + tm.t_base;
  const double2* s0 = vptr(a, tm.src[0]);
  const double2* s1 = tm.nsrc > 1 ? vptr(a, tm.src[1]) : nullptr;
  for (int s = t.r0 + warp; s < t.r1; s += EXEC_WARPS) {
    const DevSlot sl = a.slots[kp.slot0 + s];
    const double2* V = a.fac + sl.v_off;
    const double2* x0 = s0 + sl.col_off;
    const double2* x1 = s1 ? s1 + sl.col_off : nullptr;
    double2 d = make_double2(0.0, 0.0);
    constexpr int U = 4;
    for (int c0 = lane; c0 < sl.cols; c0 += 32 * U) {
      double2 vv[U], xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + 32 * u;
        const bool in = c < sl.cols;
        vv[u] = in ? ld_stream(V + c) : make_double2(0.0, 0.0);
        xv[u] = in ? ld_cg(x0 + c) : make_double2(0.0, 0.0);
        if (x1 && in) xv[u] = cadd(xv[u], ld_cg(x1 + c));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) d = cfma(vv[u], xv[u], d);
    }
    d = warp_sum(d);
    if (lane == 0) st_cg(T + s, d);
  }
}

// rows of one output block from PLR terms: thread per row,
// y_r = sum over leaves covering r of U_leaf[r, :] . t_leaf (U column-major).
__device__ void run_y_plr(const ExecArgs& a, const DevTask& t) {
  const int row = t.r0 + threadIdx.x;
  const bool act = row < t.r1;
  double2 acc = make_double2(0.0, 0.0);
  if (act && t.has_init) acc = ld_cg(vptr(a, t.init) + row);
  for (int it = 0; it < t.nterm; ++it) {
    const DevTerm tm = a.terms[t.term0 + it];
    if (!act) continue;
    const DevKernelPLR kp = a.kplr[tm.kernel];
    const double2* T = a.slot[SLOT_T] + tm.t_base;
    const DevSegment sg = a.segs[a.rowseg[kp.seg0 + row]];
    double2 at = make_double2(0.0, 0.0);
    for (int l = 0; l < sg.nleaf; ++l) {
      const DevLeaf lf = a.leaves[a.seg_leaves[sg.leaf_list0 + l]];
      const double2* U = a.fac + lf.u_off + (row - lf.row_off);
      const double2* tt = T + lf.slot0;
      int c = 0;
      for (; c + 4 <= lf.rank; c += 4) {
        double2 uv[4], tv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uv[u] = ld_stream(U + (size_t)(c + u) * lf.rows);
          tv[u] = ld_cg(tt + c + u);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) at = cfma(uv[u], tv[u], at);
      }
      for (; c < lf.rank; ++c) at = cfma(ld_stream(U + (size_t)c * lf.rows), ld_cg(tt + c), at);
    }
    acc = cfma(make_double2(tm.scale_re, tm.scale_im), at, acc);
  }
  if (!act) return;
  for (int e = 0; e < t.neye; ++e) {
    const DevEye ey = a.eyes[t.eye0 + e];
    acc = cfma(make_double2(ey.re, ey.im), ld_cg(vptr(a, ey.src) + row), acc);
  }
  if (t.has_rhs) {
    const double2 r = ld_cg(vptr(a, t.rhs) + row);
    acc.x = fma(t.rhs_coef, r.x, acc.x);
    acc.y = fma(t.rhs_coef, r.y, acc.y);
  }
  st_cg(vptr_w(a, t.out) + row, acc);
}

}  // namespace

__global__ void __launch_bounds__(EXEC_THREADS) pt_exec_kernel(ExecArgs a) {
  extern __shared__ double2 smem[];
  __shared__ int s_task;
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
      run_t_plr(a, t);
    else
      run_y_plr(a, t);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(a.ctr + t.signal, 1);
    }
  }
}

}  // namespace pt
