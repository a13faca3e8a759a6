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
// Operator data moves HBM -> shared memory with TMA bulk copies
// (cp.async.bulk.shared::cluster.global, completion on an mbarrier).  Every
// task's operator bytes are a few contiguous "pieces" (host layout: a Vt
// region per kernel and tile-major U chunks), double-buffered in two smem
// halves.  The first two pieces are issued when the task is grabbed, BEFORE
// its dependency wait: the operator never depends on the iterate, so a sweep
// level's kernels stream in while the previous level is still computing.
// After the wait the task stages its (small) vector inputs, waits for the
// pieces and computes from shared memory (FP64 FMA, fixed-order sums, no
// float atomics: repeated applies are bitwise identical).
#include "pt_device.cuh"

namespace pt {

namespace {

// slot base pointers of this launch (iteration-relative ones resolved)
__shared__ double2* s_slot[N_SLOTS];
__shared__ __align__(8) unsigned long long s_bar[2];  // one mbarrier per buffer half

__device__ __forceinline__ const double2* vptr(const VecRef& r) { return s_slot[r.slot] + r.off; }
__device__ __forceinline__ double2* vptr_w(const VecRef& r) { return s_slot[r.slot] + r.off; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// thread 0: stage one piece into a buffer half (TMA bulk copy, mbarrier tx)
__device__ __forceinline__ void issue_piece(unsigned long long* bar, double2* dst,
                                            const double2* src, uint32_t bytes) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void wait_bar(unsigned long long* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}

struct Smem {
  double2* half[2];    // operator piece buffers
  double2* src;        // staged source vector (m) / t values (MAX_TCOLS)
  double2* part;       // EXEC_THREADS partial sums
  void* meta;          // task metadata (entries / slots)
};

__device__ __forceinline__ Smem carve(double2* base, const ExecArgs& a) {
  Smem s;
  s.half[0] = base;
  s.half[1] = base + a.half_elems;
  s.src = base + 2 * a.half_elems;
  s.part = s.src + a.src_cap;
  s.meta = s.part + EXEC_THREADS;
  return s;
}

// per-CTA pipeline state (uniform across threads)
struct Pipe {
  uint32_t phase[2];
};

__device__ __forceinline__ const double2* pool_of(const ExecArgs& a, const DevTask& t) {
  return t.type == TASK_Y_DENSE ? a.dense : a.fac;
}

// thread 0 issues piece p of task t into half p % 2
__device__ __forceinline__ void issue(const ExecArgs& a, const DevTask& t, const Smem& sm, int p) {
  const DevPiece pc = a.pieces[t.piece0 + p];
  issue_piece(&s_bar[p & 1], sm.half[p & 1], pool_of(a, t) + pc.src,
              (uint32_t)pc.elems * (uint32_t)sizeof(double2));
}

__device__ __forceinline__ const double2* wait_piece(Pipe& pp, int p, const Smem& sm) {
  wait_bar(&s_bar[p & 1], pp.phase[p & 1]);
  pp.phase[p & 1] ^= 1u;
  return sm.half[p & 1];
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

// ---- metadata staging (before the dependency wait) --------------------------------

__device__ __forceinline__ void stage_meta(const ExecArgs& a, const DevTask& t, const Smem& sm) {
  if (t.type == TASK_Y_PLR) {
    DevTileEntry* ent = reinterpret_cast<DevTileEntry*>(sm.meta);
    for (int i = threadIdx.x; i < t.nent; i += EXEC_THREADS) ent[i] = a.ents[t.ent0 + i];
  } else if (t.type == TASK_T_PLR) {
    const DevTerm tm = a.terms[t.term0];
    const int32_t slot0 = a.kplr[tm.kernel].slot0;
    DevSlot* sl = reinterpret_cast<DevSlot*>(sm.meta);
    for (int q = threadIdx.x; q < t.r1 - t.r0; q += EXEC_THREADS) sl[q] = a.slots[slot0 + t.r0 + q];
  }
}

// ---- Y_DENSE: rows [r0, r1) from dense kernel terms -------------------------------
// piece p = rows r0..r1 of term p's kernel (row-major, staged in smem).
// Columns are split over the 8 warps; each warp keeps its scaled partial per
// row in smem; partials are added in warp order.
__device__ __forceinline__ void run_y_dense(const ExecArgs& a, const DevTask& t, const Smem& sm, Pipe& pp) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = a.m;
  const int nrows = t.r1 - t.r0;
  double2* part = sm.part;  // [EXEC_WARPS][DENSE_RT_MAX]
  if (lane < DENSE_RT_MAX) part[warp * DENSE_RT_MAX + lane] = make_double2(0.0, 0.0);
  __syncthreads();  // partials visible to the final sum even when there are no terms
  for (int it = 0; it < t.nterm; ++it) {
    const DevTerm tm = a.terms[t.term0 + it];
    stage_source(tm, sm.src, m);
    __syncthreads();
    const double2* K = wait_piece(pp, it, sm);
    double2 d[DENSE_RT_MAX];
#pragma unroll
    for (int k = 0; k < DENSE_RT_MAX; ++k) d[k] = make_double2(0.0, 0.0);
    for (int c = 32 * warp + lane; c < m; c += EXEC_THREADS) {
      const double2 sv = sm.src[c];
#pragma unroll
      for (int k = 0; k < DENSE_RT_MAX; ++k)
        if (k < nrows) d[k] = cfma(K[k * m + c], sv, d[k]);
    }
    const double2 sc = make_double2(tm.scale_re, tm.scale_im);
#pragma unroll
    for (int k = 0; k < DENSE_RT_MAX; ++k) {
      const double2 r = warp_sum(d[k]);
      if (lane == k && k < nrows)
        part[warp * DENSE_RT_MAX + k] = cfma(sc, r, part[warp * DENSE_RT_MAX + k]);
    }
    __syncthreads();  // buffer half and source free
    if (threadIdx.x == 0 && it + 2 < t.npiece) issue(a, t, sm, it + 2);
  }
  if ((int)threadIdx.x >= nrows) return;
  double2 v = make_double2(0.0, 0.0);
  for (int w = 0; w < EXEC_WARPS; ++w) v = cadd(v, part[w * DENSE_RT_MAX + threadIdx.x]);
  finish_row(a, t, t.r0 + threadIdx.x, v);
}

// ---- T_PLR: t = scale * Vt (x_a [+ x_b]) for a slot range ----------------------------
// The Vt rows of the task are one piece (contiguous in the Vt region); warp per
// Vt row, lanes across columns, everything from smem.  The term's scale is
// folded into t so the Y phase is a plain U t sum.
__device__ __forceinline__ void run_t_plr(const ExecArgs& a, const DevTask& t, const Smem& sm, Pipe& pp) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const DevTerm tm = a.terms[t.term0];
  double2* T = s_slot[SLOT_T] + tm.t_base;
  stage_source(tm, sm.src, a.m);
  __syncthreads();
  const DevSlot* sl = reinterpret_cast<const DevSlot*>(sm.meta);
  const double2 sc = make_double2(tm.scale_re, tm.scale_im);
  for (int p = 0; p < t.npiece; ++p) {
    const DevPiece pc = a.pieces[t.piece0 + p];
    const double2* buf = wait_piece(pp, p, sm);
    for (int q = pc.f0 + warp; q < pc.f1; q += EXEC_WARPS) {
      const DevSlot d = sl[q];
      const double2* V = buf + (d.v_off - pc.src);
      const double2* x = sm.src + d.col_off;
      double2 r = make_double2(0.0, 0.0);
      for (int c = lane; c < d.cols; c += 32) r = cfma(V[c], x[c], r);
      r = warp_sum(r);
      if (lane == 0) st_cg(T + t.r0 + q, cmul(sc, r));
    }
    __syncthreads();
    if (threadIdx.x == 0 && p + 2 < t.npiece) issue(a, t, sm, p + 2);
  }
}

// ---- Y_PLR: one PLR_TILE-row tile ---------------------------------------------------
// y_r = sum over the task's flat (entry, rank column) list of U[r, c] t[c].
// Thread = (row r = tid % 16, column group g = tid / 16): group g takes flat
// columns f = g (mod 16) in ascending order; the 16 partial sums per row are
// added in group order.  U pieces and the t values are read from smem.
__device__ __forceinline__ void run_y_plr(const ExecArgs& a, const DevTask& t, const Smem& sm, Pipe& pp) {
  constexpr int G = EXEC_THREADS / PLR_TILE;  // 16 column groups
  const int r = threadIdx.x % PLR_TILE, g = threadIdx.x / PLR_TILE;
  const DevTileEntry* ent = reinterpret_cast<const DevTileEntry*>(sm.meta);
  // t values of every flat column (produced by this level's T tasks)
  double2* ts = sm.src;
  {
    const double2* T = s_slot[SLOT_T];
    int e = 0;
    for (int f = threadIdx.x; f < t.ncol; f += EXEC_THREADS) {
      while (e + 1 < t.nent && f >= ent[e + 1].pre) ++e;
      ts[f] = ld_cg(T + ent[e].t0 + (f - ent[e].pre));
    }
  }
  __syncthreads();
  double2 acc = make_double2(0.0, 0.0);
  for (int p = 0; p < t.npiece; ++p) {
    const DevPiece pc = a.pieces[t.piece0 + p];
    const double2* buf = wait_piece(pp, p, sm);
    int e = pc.e0;
    // first column of this group inside the piece
    int f = pc.f0 + ((g - pc.f0) % G + G) % G;
    for (; f < pc.f1; f += G) {
      while (e + 1 < t.nent && f >= ent[e + 1].pre) ++e;
      const DevTileEntry en = ent[e];
      if (r >= en.lo && r < en.hi) {
        const int c = f - en.pre;
        const double2 u = buf[en.u0 + (int64_t)c * en.stride - pc.src + (r - en.lo)];
        acc = cfma(u, ts[f], acc);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && p + 2 < t.npiece) issue(a, t, sm, p + 2);
  }
  sm.part[g * PLR_TILE + r] = acc;
  __syncthreads();
  if ((int)threadIdx.x >= PLR_TILE || t.r0 + (int)threadIdx.x >= t.r1) return;
  double2 v = make_double2(0.0, 0.0);
#pragma unroll
  for (int q = 0; q < G; ++q) v = cadd(v, sm.part[q * PLR_TILE + threadIdx.x]);
  finish_row(a, t, t.r0 + threadIdx.x, v);
}

}  // namespace

// thread 0: asynchronous copy of a task descriptor into smem (cp.async)
__device__ __forceinline__ void fetch_task(DevTask* dst, const DevTask* src) {
  static_assert(sizeof(DevTask) % 16 == 0, "DevTask must be a multiple of 16 bytes");
  const char* s = reinterpret_cast<const char*>(src);
  const uint32_t d = smem_u32(dst);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(DevTask) / 16); ++i)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 16 * i), "l"(s + 16 * i)
                 : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(EXEC_THREADS, 3) pt_exec_kernel(ExecArgs a) {
  extern __shared__ __align__(128) double2 smem[];
  __shared__ __align__(16) DevTask s_desc[2];  // current / next task descriptors
  __shared__ int s_q[2];
  __shared__ int s_stop;
  if (a.stop) {
    if (threadIdx.x == 0) s_stop = *((volatile const int*)a.stop);
    __syncthreads();
    if (s_stop) return;
  }
  if (threadIdx.x < N_SLOTS) {
    double2* p = a.slot[threadIdx.x];
    if (a.iter && (threadIdx.x == SLOT_IN || threadIdx.x == SLOT_OUT)) {
      const int64_t j = *((volatile const int*)a.iter) + (threadIdx.x == SLOT_OUT ? 1 : 0);
      p = a.vbase + j * a.vstride;
    }
    s_slot[threadIdx.x] = p;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[i])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int q0 = atomicAdd(a.head, 1);
    s_q[0] = q0;
    if (q0 < a.n_tasks) fetch_task(&s_desc[0], a.tasks + q0);
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  const Smem sm = carve(smem, a);
  Pipe pp;
  pp.phase[0] = pp.phase[1] = 0;
  int b = 0;
  for (;;) {
    const int q = s_q[b];
    if (q >= a.n_tasks) break;
    const DevTask& t = s_desc[b];
    int q_next = 0;
    unsigned long long t_grab = 0, t_ready = 0;
    // grab the next task now; its index is needed only after the wait below
    if (threadIdx.x == 0) {
      q_next = atomicAdd(a.head, 1);
      if (a.trace) t_grab = globaltimer();
      // prepare: start the operator copies (input independent)
      for (int p = 0; p < t.npiece && p < 2; ++p) issue(a, t, sm, p);
    }
    stage_meta(a, t, sm);
    // wait for the producers of the inputs; then prefetch the next descriptor
    if (threadIdx.x == 0) {
      for (int w = 0; w < t.nwait; ++w) {
        const DevWait dw = a.waits[t.wait0 + w];
        while (ld_acquire(a.ctr + dw.ctr) < dw.val) __nanosleep(32);
      }
      if (a.trace) t_ready = globaltimer();
      s_q[b ^ 1] = q_next;
      if (q_next < a.n_tasks) fetch_task(&s_desc[b ^ 1], a.tasks + q_next);
    }
    __syncthreads();
    if (t.type == TASK_Y_DENSE)
      run_y_dense(a, t, sm, pp);
    else if (t.type == TASK_T_PLR)
      run_t_plr(a, t, sm, pp);
    else
      run_y_plr(a, t, sm, pp);
    if (threadIdx.x == 0) asm volatile("cp.async.wait_all;" ::: "memory");
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
    b ^= 1;
  }
}

}  // namespace pt
