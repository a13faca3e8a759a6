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
// A task runs in three phases:
//   prepare  -- before its inputs are ready: issue TMA bulk prefetches
//               (cp.async.bulk.prefetch.L2) of the kernel data it will
//               stream and stage its metadata in smem.  Kernel data never
//               depends on the iterate, so HBM streaming of a sweep level
//               overlaps the previous level's dependency chain.
//   wait     -- thread 0 acquires the producer counters.
//   compute  -- 16-byte complex loads (now mostly L2 hits), FP64 FMA,
//               fixed-order reductions.
//
// Kernel data is read with ld.global.nc.L1::no_allocate; vectors written
// during the launch are read through L2 (ld.cg).  Each output element is
// produced by one CTA in a fixed order, so repeated applies are bitwise
// identical (no float atomics).
#include "pt_device.cuh"

namespace pt {

namespace {

// slot base pointers of this launch (iteration-relative ones resolved), in smem
__shared__ double2* s_slot[N_SLOTS];

__device__ __forceinline__ const double2* vptr(const VecRef& r) { return s_slot[r.slot] + r.off; }
__device__ __forceinline__ double2* vptr_w(const VecRef& r) { return s_slot[r.slot] + r.off; }

struct Smem {
  double2* src;        // m: staged source vector
  double2* part;       // EXEC_THREADS: partial sums
  DevTileEntry* ent;   // MAX_TILE_ENTRIES: task metadata (Y_PLR entries / T slots)
};

__device__ __forceinline__ Smem carve(double2* base, int m) {
  Smem s;
  s.src = base;
  s.part = base + m;
  s.ent = reinterpret_cast<DevTileEntry*>(base + m + EXEC_THREADS);
  return s;
}

// stage x_a [+ x_b] (length m) into smem
__device__ __forceinline__ void stage_source(const DevTerm& tm, double2* s, int m) {
  const double2* s0 = vptr(tm.src[0]);
  if (tm.nsrc > 1) {
    const double2* s1 = vptr(tm.src[1]);
    for (int c = threadIdx.x; c < m; c += EXEC_THREADS) s[c] = cadd(ld_cg(s0 + c), ld_cg(s1 + c));
  } else {
    for (int c = threadIdx.x; c < m; c += EXEC_THREADS) s[c] = ld_cg(s0 + c);
  }
}

// final per-row epilogue: init + partial sum + eyes + rhs -> out
__device__ __forceinline__ void finish_row(const ExecArgs& a, const DevTask& t, int row,
                                           double2 v) {
  if (t.has_init) v = cadd(ld_cg(vptr(t.init) + row), v);
  for (int e = 0; e < t.neye; ++e) {
    const DevEye ey = a.eyes[t.eye0 + e];
    v = cfma(make_double2(ey.re, ey.im), ld_cg(vptr(ey.src) + row), v);
  }
  if (t.has_rhs) {
    const double2 r = ld_cg(vptr(t.rhs) + row);
    v.x = fma(t.rhs_coef, r.x, v.x);
    v.y = fma(t.rhs_coef, r.y, v.y);
  }
  st_cg(vptr_w(t.out) + row, v);
}

// ---- Y_DENSE ------------------------------------------------------------------

__device__ void prepare_y_dense(const ExecArgs& a, const DevTask& t) {
  if ((int)threadIdx.x < t.nterm) {
    const DevTerm tm = a.terms[t.term0 + threadIdx.x];
    const int m = a.m;
    prefetch_l2(a.dense + ((size_t)tm.kernel * m + t.r0) * m,
                (uint32_t)((t.r1 - t.r0) * (size_t)m * sizeof(double2)));
  }
}

// Up to DENSE_RT_MAX rows from dense kernel terms.  Columns are split over
// the 8 warps (warp w takes columns 32w + lane + 256 i); each warp keeps its
// scaled partial per row in smem and the partials are added in warp order.
__device__ void run_y_dense(const ExecArgs& a, const DevTask& t, const Smem& sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = a.m;
  const int nrows = t.r1 - t.r0;
  double2* part = sm.part;  // [EXEC_WARPS][DENSE_RT_MAX]
  if (lane < DENSE_RT_MAX) part[warp * DENSE_RT_MAX + lane] = make_double2(0.0, 0.0);
  for (int it = 0; it < t.nterm; ++it) {
    const DevTerm tm = a.terms[t.term0 + it];
    __syncthreads();
    stage_source(tm, sm.src, m);
    __syncthreads();
    const double2* K = a.dense + ((size_t)tm.kernel * m + t.r0) * m;
    double2 d[DENSE_RT_MAX];
#pragma unroll
    for (int k = 0; k < DENSE_RT_MAX; ++k) d[k] = make_double2(0.0, 0.0);
    for (int c = 32 * warp + lane; c < m; c += EXEC_THREADS) {
      double2 kv[DENSE_RT_MAX];
#pragma unroll
      for (int k = 0; k < DENSE_RT_MAX; ++k)
        kv[k] = k < nrows ? ld_stream(K + (size_t)k * m + c) : make_double2(0.0, 0.0);
      const double2 sv = sm.src[c];
#pragma unroll
      for (int k = 0; k < DENSE_RT_MAX; ++k) d[k] = cfma(kv[k], sv, d[k]);
    }
    const double2 sc = make_double2(tm.scale_re, tm.scale_im);
#pragma unroll
    for (int k = 0; k < DENSE_RT_MAX; ++k) {
      const double2 r = warp_sum(d[k]);
      if (lane == k && k < nrows)
        part[warp * DENSE_RT_MAX + k] = cfma(sc, r, part[warp * DENSE_RT_MAX + k]);
    }
  }
  __syncthreads();
  if ((int)threadIdx.x >= nrows) return;
  double2 v = make_double2(0.0, 0.0);
  for (int w = 0; w < EXEC_WARPS; ++w) v = cadd(v, part[w * DENSE_RT_MAX + threadIdx.x]);
  finish_row(a, t, t.r0 + threadIdx.x, v);
}

// ---- T_PLR ----------------------------------------------------------------------

__device__ void prepare_t_plr(const ExecArgs& a, const DevTask& t, const Smem& sm) {
  const DevTerm tm = a.terms[t.term0];
  const int32_t slot0 = a.kplr[tm.kernel].slot0;
  DevSlot* sl = reinterpret_cast<DevSlot*>(sm.ent);
  for (int q = threadIdx.x; q < t.r1 - t.r0; q += EXEC_THREADS) {
    const DevSlot d = a.slots[slot0 + t.r0 + q];
    sl[q] = d;
    prefetch_l2(a.fac + d.v_off, (uint32_t)d.cols * sizeof(double2));
  }
}

// t = scale * Vt (x_a [+ x_b]) for a slot range of one PLR term: source staged
// in smem, warp per Vt row (two rows in flight per warp), lanes across
// columns.  The term's scale is folded into t so Y is a plain U t sum.
__device__ void run_t_plr(const ExecArgs& a, const DevTask& t, const Smem& sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = a.m;
  const DevTerm tm = a.terms[t.term0];
  double2* T = s_slot[SLOT_T] + tm.t_base;
  stage_source(tm, sm.src, m);
  __syncthreads();
  const DevSlot* sl = reinterpret_cast<const DevSlot*>(sm.ent);
  const double2 sc = make_double2(tm.scale_re, tm.scale_im);
  const int ns = t.r1 - t.r0;
  for (int q = warp; q < ns; q += 2 * EXEC_WARPS) {
    const int q2 = q + EXEC_WARPS;
    const DevSlot d1 = sl[q];
    const bool has2 = q2 < ns;
    const DevSlot d2 = has2 ? sl[q2] : d1;
    const int n2 = has2 ? d2.cols : 0;
    const double2* V1 = a.fac + d1.v_off;
    const double2* V2 = a.fac + d2.v_off;
    const double2* x1 = sm.src + d1.col_off;
    const double2* x2 = sm.src + d2.col_off;
    double2 r1 = make_double2(0.0, 0.0), r2 = make_double2(0.0, 0.0);
    const int cmax = max(d1.cols, n2);
    constexpr int U = 4;
    for (int c0 = lane; c0 < cmax; c0 += 32 * U) {
      double2 v1[U], v2[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + 32 * u;
        v1[u] = c < d1.cols ? ld_stream(V1 + c) : make_double2(0.0, 0.0);
        v2[u] = c < n2 ? ld_stream(V2 + c) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + 32 * u;
        if (c < d1.cols) r1 = cfma(v1[u], x1[c], r1);
        if (c < n2) r2 = cfma(v2[u], x2[c], r2);
      }
    }
    r1 = warp_sum(r1);
    r2 = warp_sum(r2);
    if (lane == 0) {
      st_cg(T + t.r0 + q, cmul(sc, r1));
      if (has2) st_cg(T + t.r0 + q2, cmul(sc, r2));
    }
  }
}

// ---- Y_PLR ----------------------------------------------------------------------

// Stage the task's flat tile entries (host-built: t0 absolute, prefix
// column counts) in smem and prefetch their U column segments into L2.
__device__ void prepare_y_plr(const ExecArgs& a, const DevTask& t, const Smem& sm) {
  for (int i = threadIdx.x; i < t.nent; i += EXEC_THREADS) {
    const DevTileEntry e = a.ents[t.ent0 + i];
    sm.ent[i] = e;
    const uint32_t bytes = (uint32_t)(e.hi - e.lo) * sizeof(double2);
    for (int c = 0; c < e.rank; ++c) prefetch_l2(a.fac + e.u0 + (int64_t)c * e.stride, bytes);
  }
}

// One PLR_TILE-row tile of an output block: y_r = sum over the staged
// entries of U_leaf[r, :] t_leaf.  Lane = row (U is column-major: a warp
// reads up to 32 consecutive rows of one rank column, contiguous bytes); the
// (entry, column) pairs are dealt round-robin to the 8 warps, and the 8
// partial sums per row are added in warp order.
__device__ void run_y_plr(const ExecArgs& a, const DevTask& t, const Smem& sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = t.r0 + lane;
  const double2* T = s_slot[SLOT_T];
  const int count = t.nent;
  const int ncol = count ? sm.ent[count - 1].pre + sm.ent[count - 1].rank : 0;
  double2 acc = make_double2(0.0, 0.0);
  constexpr int B = 8;  // independent columns in flight per warp
  int e = 0;
  for (int f0 = warp; f0 < ncol; f0 += B * EXEC_WARPS) {
    double2 uv[B], tv[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int f = f0 + b * EXEC_WARPS;
      uv[b] = make_double2(0.0, 0.0);
      tv[b] = make_double2(0.0, 0.0);
      if (f < ncol) {
        while (e + 1 < count && f >= sm.ent[e + 1].pre) ++e;
        const DevTileEntry en = sm.ent[e];
        const int c = f - en.pre;
        if (lane >= en.lo && lane < en.hi)
          uv[b] = ld_stream(a.fac + en.u0 + (int64_t)c * en.stride + (lane - en.lo));
        tv[b] = ld_cg(T + en.t0 + c);
      }
    }
#pragma unroll
    for (int b = 0; b < B; ++b) acc = cfma(uv[b], tv[b], acc);
  }
  sm.part[warp * 32 + lane] = acc;
  __syncthreads();
  if (warp != 0 || row >= t.r1) return;
  double2 v = make_double2(0.0, 0.0);
#pragma unroll
  for (int w = 0; w < EXEC_WARPS; ++w) v = cadd(v, sm.part[w * 32 + lane]);
  finish_row(a, t, row, v);
}

}  // namespace

__global__ void __launch_bounds__(EXEC_THREADS, 3) pt_exec_kernel(ExecArgs a) {
  extern __shared__ double2 smem[];
  __shared__ int s_task;
  if (a.stop) {
    if (threadIdx.x == 0) s_task = *((volatile const int*)a.stop);
    __syncthreads();
    if (s_task) return;
    __syncthreads();
  }
  if (threadIdx.x < N_SLOTS) {
    double2* p = a.slot[threadIdx.x];
    if (a.iter && (threadIdx.x == SLOT_IN || threadIdx.x == SLOT_OUT)) {
      const int64_t j = *((volatile const int*)a.iter) + (threadIdx.x == SLOT_OUT ? 1 : 0);
      p = a.vbase + j * a.vstride;
    }
    s_slot[threadIdx.x] = p;
  }
  __syncthreads();
  const Smem sm = carve(smem, a.m);
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(a.head, 1);
    __syncthreads();
    const int q = s_task;
    if (q >= a.n_tasks) return;
    const DevTask t = a.tasks[q];
    unsigned long long t_grab = 0, t_ready = 0;
    if (a.trace && threadIdx.x == 0) t_grab = globaltimer();
    // prepare: prefetch kernel data + stage metadata (independent of the inputs)
    if (t.type == TASK_Y_DENSE)
      prepare_y_dense(a, t);
    else if (t.type == TASK_T_PLR)
      prepare_t_plr(a, t, sm);
    else
      prepare_y_plr(a, t, sm);
    // wait for the producers of the inputs
    if (threadIdx.x == 0) {
      for (int w = 0; w < t.nwait; ++w) {
        const DevWait dw = a.waits[t.wait0 + w];
        while (ld_acquire(a.ctr + dw.ctr) < dw.val) __nanosleep(32);
      }
      if (a.trace) t_ready = globaltimer();
    }
    __syncthreads();
    if (t.type == TASK_Y_DENSE)
      run_y_dense(a, t, sm);
    else if (t.type == TASK_T_PLR)
      run_t_plr(a, t, sm);
    else
      run_y_plr(a, t, sm);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(a.ctr + t.signal, 1);
      if (a.trace) {
        unsigned long long* tr = a.trace + 4 * (size_t)q;
        tr[0] = t_grab;
        tr[1] = t_ready;
        tr[2] = globaltimer();
        tr[3] = smid();
      }
    }
  }
}

}  // namespace pt
