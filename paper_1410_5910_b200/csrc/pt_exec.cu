// Persistent dataflow executor for interface-operator programs.
//
// One launch runs a whole program: an A-apply, a preconditioner apply of
// n_it Gauss-Seidel sweeps, or a fused A -> M GMRES iteration.  The host
// compiles the program into a task DAG whose queue order is topological.
// Tasks wait on the counters of the producer groups they read and bump
// their own group's counter.  The launch is cooperative: every CTA is
// resident, so a waiting task always has a running producer.
//
// Each CTA is warp-specialised.  Three producer warps (EXEC_PRODUCERS) own
// one task slot each and take the CTA's tasks in rotation (grabbed one at a
// time, in order); per task a producer warp:
//   - bulk-copies the task's metadata blob (descriptor, operator pieces,
//     terms, eyes, waits, per-column items) into its slot: one TMA copy;
//   - issues the task's operator pieces into the CTA's smem ring with TMA
//     bulk copies (cp.async.bulk, mbarrier complete_tx) as far as the ring
//     allows -- BEFORE the dependency wait, when it is this task's turn;
//   - waits for the dependency counters;
//   - stages the vector inputs (source slice, t values, term sources,
//     epilogue rows) with TMA bulk copies, all in flight at once;
//   - hands the slot to the consumers (mbarrier), then streams the task's
//     remaining pieces and passes the ring to the next task.
// With three producer warps the metadata, dependency and staging latency of
// tasks n+1 and n+2 overlaps the consumers' work on task n, and the operator
// stream of the next sweep level overlaps the current level's dependency
// chain.  The 16 consumer warps compute from shared memory (FP64 FMA,
// fixed-order sums), release ring stages and slots through mbarriers and
// write the outputs; the slot's producer warp then signals the counter
// (red.release.gpu).  No float atomics anywhere: every output element is
// produced by one CTA in a fixed order, so repeated applies are bitwise
// identical.  The last CTA out resets the counters for the next launch.
#include "pt_device.cuh"

namespace pt {

namespace {

constexpr int CONSUMERS = EXEC_CONSUMERS;  // 512 threads, 16 warps

// ---- checked build (PT_CHECK, see pt_device.cuh) --------------------------------
#if PT_CHECK
__shared__ long long* s_errp;
__device__ __noinline__ void chk_fail(int code, long long q, long long val) {
  if (s_errp && atomicCAS((unsigned long long*)s_errp, 0ull, (unsigned long long)code) == 0ull) {
    s_errp[1] = q;
    s_errp[2] = val;
    __threadfence_system();
  }
  __trap();
}
#define CHK(cond, code, q, val)                      \
  do {                                               \
    if (!(cond)) chk_fail((code), (q), (long long)(val)); \
  } while (0)
// spin-loop watchdog: ~4e9 cycles (~2 s) in one wait is a hang
#define SPIN_DECL const long long spin0_ = clock64()
#define SPIN_CHECK(q) CHK(clock64() - spin0_ < 4000000000ll, CHK_HANG, (q), 0)
#else
#define CHK(cond, code, q, val) \
  do {                          \
  } while (0)
#define SPIN_DECL \
  do {            \
  } while (0)
#define SPIN_CHECK(q) \
  do {                \
  } while (0)
#endif
constexpr int CWARPS = CONSUMERS / 32;

__shared__ double2* s_slot[N_SLOTS];
__shared__ __align__(8) unsigned long long s_full[EXEC_MAX_STAGES];   // piece landed (tx)
__shared__ __align__(8) unsigned long long s_empty[EXEC_MAX_STAGES];  // piece consumed
__shared__ __align__(8) unsigned long long s_tfull[EXEC_TSLOTS];      // slot handed over
__shared__ __align__(8) unsigned long long s_tempty[EXEC_TSLOTS];     // slot released
__shared__ __align__(8) unsigned long long s_meta[EXEC_TSLOTS];       // blob landed (tx)
__shared__ __align__(8) unsigned long long s_stg[EXEC_TSLOTS];        // vectors landed (tx)
__shared__ volatile int s_grab_turn;     // slot use whose task may be grabbed next
// Ring positions are reserved per slot use, in use order, as soon as the
// task's piece count is known: a use's pieces may then be issued before the
// previous use has issued all of its own (each position waits only for the
// stage's previous occupant to be consumed).
__shared__ volatile int s_resv_turn;     // slot use that reserves positions next
__shared__ volatile uint32_t s_next_pos; // first unreserved ring position
// Ring positions fully consumed (a lower bound: updated by the consumers at
// the end of every task).  A stage's empty barrier is tested by parity, which
// only tells apart two consecutive phases; a producer therefore looks at the
// first positions of its use only while pos < s_consumed + 2 * n_stages (then
// the phase of pos - n_stages is the current or the previous one), see
// in_window.  Without the bound a producer several uses ahead (long tasks, or
// more than two task slots) could read an older phase as complete.
__shared__ volatile uint32_t s_consumed;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bar_init(unsigned long long* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bar_expect(unsigned long long* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool bar_test(unsigned long long* b, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(done)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ void bar_wait(unsigned long long* b, uint32_t parity) {
  uint32_t done = 0;
  SPIN_DECL;
  while (!done) {
    SPIN_CHECK(-1);
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  }
}
// TMA bulk copy global -> this CTA's shared memory, completing on mbarrier b
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes,
                                          unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(CONSUMERS) : "memory");
}

// ---- shared-memory layout -------------------------------------------------------

// A task slot: [metadata blob][staged vectors][epilogue rows][coefficients]
// [vector pointers].  Blob sections are located by the descriptor's offsets.
struct Slot {
  char* blob;
  double2* vec;         // staged vector inputs (source slice / t values / term sources)
  double2* epi;         // epilogue source rows: [k * EXEC_EPI + row], k = init, eyes, rhs
  double2* coef;        // term scales [0, EXEC_TERMS), eye coefficients after them
  const double2** src;  // vector pointers: term sources [2 * term + s], then
                        // epilogue rows [2 * EXEC_TERMS + k]
  __device__ __forceinline__ const DevTask& desc() const {
    return *reinterpret_cast<const DevTask*>(blob);
  }
  __device__ __forceinline__ const DevPiece* pieces() const {
    return reinterpret_cast<const DevPiece*>(blob + desc().piece0);
  }
  __device__ __forceinline__ const DevTerm* terms() const {
    return reinterpret_cast<const DevTerm*>(blob + desc().term0);
  }
  __device__ __forceinline__ const DevEye* eyes() const {
    return reinterpret_cast<const DevEye*>(blob + desc().eye0);
  }
  __device__ __forceinline__ const DevWait* waits() const {
    return reinterpret_cast<const DevWait*>(blob + desc().wait0);
  }
  __device__ __forceinline__ const DevItem* items() const {
    return reinterpret_cast<const DevItem*>(blob + desc().item0);
  }
  __device__ __forceinline__ const DevRun* runs() const {
    return reinterpret_cast<const DevRun*>(blob + desc().run0);
  }
  __device__ __forceinline__ const DevSrcRun* sruns() const {
    return reinterpret_cast<const DevSrcRun*>(blob + desc().srun0);
  }
};

// computed on use (arrays of pointers would be indexed dynamically and live
// on the stack)
struct Layout {
  char* base;
  int64_t stage_bytes, slot_bytes, blob_cap, vec_cap;
  int n_stages;
  int n_slots;  // task slots in use (<= EXEC_TSLOTS)
  __device__ __forceinline__ double2* stage(int s) const {
    return reinterpret_cast<double2*>(base + (size_t)s * stage_bytes);
  }
  __device__ __forceinline__ Slot slot(int k) const {
    char* q = base + (size_t)n_stages * stage_bytes + (size_t)k * slot_bytes;
    Slot sl;
    sl.blob = q;
    q += blob_cap;
    sl.vec = reinterpret_cast<double2*>(q);
    q += (size_t)vec_cap * sizeof(double2);
    sl.epi = reinterpret_cast<double2*>(q);
    q += EXEC_EPI * EXEC_EPI_SRC * sizeof(double2);
    sl.coef = reinterpret_cast<double2*>(q);
    q += (EXEC_TERMS + EXEC_EYES) * sizeof(double2);
    sl.src = reinterpret_cast<const double2**>(q);
    return sl;
  }
  __device__ __forceinline__ double2* part() const {
    return reinterpret_cast<double2*>(base + (size_t)n_stages * stage_bytes +
                                      (size_t)n_slots * (size_t)slot_bytes);
  }
};

__device__ __forceinline__ Layout carve(double2* base, const ExecArgs& a) {
  Layout L;
  L.base = reinterpret_cast<char*>(base);
  L.stage_bytes = a.half_elems * (int64_t)sizeof(double2);
  L.slot_bytes = a.slot_bytes;
  L.blob_cap = a.blob_cap;
  L.vec_cap = a.src_cap;
  L.n_stages = a.n_stages;
  L.n_slots = a.n_slots;
  return L;
}

__device__ __forceinline__ const double2* vptr(const VecRef& r) { return s_slot[r.slot] + r.off; }
__device__ __forceinline__ double2* vptr_w(const VecRef& r) { return s_slot[r.slot] + r.off; }

// trace words of queue index q: 0 grab, 1 ready, 2 done, 3 smid | cta << 16,
// 4 consumer start, 5 staged, 6..13 piece p landed (consumer), 14..21 piece p
// issued (producer), 22/23 consumer cycles waiting for pieces / in barriers
__device__ __forceinline__ void trace_mark(const ExecArgs& a, int q, int k) {
  if (a.trace)
    a.trace[EXEC_TRACE * (size_t)q + k] =
        k == 3 ? (unsigned long long)smid() | ((unsigned long long)blockIdx.x << 16) : globaltimer();
}

// ---- producers (warps 8, 9) ---------------------------------------------------------

// lane 0: issue piece p of the slot's task into ring position pos
__device__ __forceinline__ void issue_piece(const ExecArgs& a, const Layout& L, const Slot& sl,
                                            int q, int p, uint32_t pos) {
  const DevPiece& pc = sl.pieces()[p];
  const int s = pos % (uint32_t)L.n_stages;
  const uint32_t bytes = (uint32_t)(pc.elems + pc.elems2) * (uint32_t)sizeof(double2);
  CHK(pc.elems > 0 && pc.elems2 >= 0 && pc.elems + pc.elems2 <= a.half_elems, CHK_PIECE_SIZE, q, pc.elems);
  CHK(pc.elems2 == 0 || (pc.src2 >= 0 && pc.src2 + pc.elems2 <= a.fac_elems), CHK_PIECE_RANGE, q, pc.src2);
  CHK(pc.src >= 0 && pc.src + pc.elems <=
                         (sl.desc().type == TASK_Y_DENSE ? a.dense_elems : a.fac_elems),
      CHK_PIECE_RANGE, q, pc.src);
  const double2* src = (sl.desc().type == TASK_Y_DENSE ? a.dense : a.fac) + pc.src;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  bar_expect(&s_full[s], bytes);
  bulk_copy(L.stage(s), src, (uint32_t)pc.elems * (uint32_t)sizeof(double2), &s_full[s]);
  if (pc.elems2 > 0)  // the second range (next term's columns) right behind the first
    bulk_copy(L.stage(s) + pc.elems, a.fac + pc.src2, (uint32_t)pc.elems2 * (uint32_t)sizeof(double2),
              &s_full[s]);
  if (p < 8) trace_mark(a, q, 14 + p);
}

// The parity test of position pos (waiting for the consumption of pos - ns)
// is valid once pos - ns has been issued: its issuer waited for pos - 2 ns.
// A use issues its own positions in order, so only the first ns positions
// of a use (pos - ns issued by an earlier use, perhaps not yet) need the
// window bound pos < s_consumed + 2 ns; later ones never wait on their own
// task's consumption (a task may hold any number of pieces).
__device__ __forceinline__ bool in_window(uint32_t pos, uint32_t pos0, uint32_t ns) {
  return pos >= pos0 + ns || pos < s_consumed + 2 * ns;
}

// lane 0: is the stage of ring position pos free (its previous occupant,
// position pos - n_stages, consumed)?
__device__ __forceinline__ bool stage_free(const Layout& L, uint32_t pos, uint32_t pos0) {
  const uint32_t ns = (uint32_t)L.n_stages;
  if (pos < ns) return true;
  if (!in_window(pos, pos0, ns)) return false;
  return bar_test(&s_empty[pos % ns], ((pos / ns) - 1) & 1);
}

// Term scales, eye coefficients and the vector pointers the staging
// dereferences, from the blob (all lanes; no global memory).
__device__ __forceinline__ void parse_meta(const DevTask& t, const Slot& sl, int lane) {
  if (lane < t.nterm) {
    const DevTerm& tm = sl.terms()[lane];
    sl.coef[lane] = make_double2(tm.scale_re, tm.scale_im);
    sl.src[2 * lane] = vptr(tm.src[0]);
    sl.src[2 * lane + 1] = tm.nsrc > 1 ? vptr(tm.src[1]) : nullptr;
  }
  const int e0 = t.has_init ? 1 : 0;
  if (lane < t.neye) {
    const DevEye& ey = sl.eyes()[lane];
    sl.coef[EXEC_TERMS + lane] = make_double2(ey.re, ey.im);
    sl.src[2 * EXEC_TERMS + e0 + lane] = vptr(ey.src);
  }
  if (lane == 0) {
    if (t.has_init) sl.src[2 * EXEC_TERMS] = vptr(t.init);
    if (t.has_rhs) sl.src[2 * EXEC_TERMS + e0 + t.neye] = vptr(t.rhs);
  }
}

// The vector inputs of task t, after its dependencies (all 32 lanes): TMA
// bulk copies of contiguous ranges (source slices, t-value runs, epilogue
// rows) completing on the slot's staging barrier, all in flight at once.  A
// merged term's second source lands right after the first; the consumers add
// it in place when they start the task (x_a + x_b, as the reference sums
// before applying the kernel; dense Y_DENSE terms are added here).
__device__ __forceinline__ void stage_vectors(const ExecArgs& a, const DevTask& t, const Slot& sl,
                                              int k, int& n_staged, int lane) {
  const int nrows = t.r1 - t.r0;
  const int nk = t.type == TASK_T_PLR ? 0 : (t.has_init ? 1 : 0) + t.neye + (t.has_rhs ? 1 : 0);
  const int m = a.m;
  uint32_t bytes = 0;  // total, for the barrier's transaction count
  if (t.type == TASK_T_PLR) {
    bytes = (uint32_t)(t.c1 - t.c0) * (sl.src[1] ? 2u : 1u);
  } else if (t.type == TASK_Y_PLR) {
    bytes = (uint32_t)(t.nitem + t.ndense2);
  } else {
    for (int it = 0; it < t.nterm; ++it) bytes += (uint32_t)m * (sl.src[2 * it + 1] ? 2u : 1u);
  }
  CHK(bytes <= (uint32_t)a.src_cap, CHK_STAGE_VEC, t.q, bytes);
  CHK(nk == 0 || (nrows <= EXEC_EPI && nk <= EXEC_EPI_SRC), CHK_EPI_ROWS, t.q, nrows);
  bytes = (bytes + (uint32_t)(nk * nrows)) * (uint32_t)sizeof(double2);
  if (bytes == 0) return;
  const uint32_t phase = (uint32_t)(n_staged++ & 1);
  // sources written by other CTAs (generic proxy) are read by the TMA
  asm volatile("fence.proxy.async.global;" ::: "memory");
  if (lane == 0) {
    asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&s_stg[k])),
                 "r"(bytes)
                 : "memory");
  }
  __syncwarp();
  if (t.type == TASK_T_PLR) {
    const uint32_t nb = (uint32_t)(t.c1 - t.c0) * (uint32_t)sizeof(double2);
    if (lane == 0) bulk_copy(sl.vec, sl.src[0] + t.c0, nb, &s_stg[k]);
    if (lane == 1 && sl.src[1]) bulk_copy(sl.vec + (t.c1 - t.c0), sl.src[1] + t.c0, nb, &s_stg[k]);
  } else if (t.type == TASK_Y_PLR) {
    const double2* T = s_slot[SLOT_T];
    const DevRun* runs = sl.runs();
    for (int i = lane; i < t.nrun; i += 32) {
      const DevRun r = runs[i];
      CHK(r.f >= 0 && r.f + r.n <= t.nitem && r.t >= 0 && r.t + r.n <= a.t_elems, CHK_SLOT_T, t.q, r.t);
      bulk_copy(sl.vec + r.f, T + r.t, (uint32_t)r.n * (uint32_t)sizeof(double2), &s_stg[k]);
    }
    const DevSrcRun* sr = sl.sruns();  // dense leaves: source columns (both sources)
    for (int i = lane; i < t.nsrun; i += 32) {
      const DevSrcRun r = sr[i];
      const uint32_t nb = (uint32_t)r.n * (uint32_t)sizeof(double2);
      bulk_copy(sl.vec + r.f, sl.src[2 * r.term] + r.col, nb, &s_stg[k]);
      if (sl.src[2 * r.term + 1])
        bulk_copy(sl.vec + t.nitem + r.b_off, sl.src[2 * r.term + 1] + r.col, nb, &s_stg[k]);
    }
  } else {
    for (int i = lane; i < 2 * t.nterm; i += 32)
      if (const double2* src = sl.src[i])
        bulk_copy(sl.vec + i * m, src, (uint32_t)m * (uint32_t)sizeof(double2), &s_stg[k]);
  }
  if (lane < nk)  // epilogue source rows: init, eyes, rhs
    bulk_copy(sl.epi + lane * EXEC_EPI, sl.src[2 * EXEC_TERMS + lane] + t.r0,
              (uint32_t)nrows * (uint32_t)sizeof(double2), &s_stg[k]);
  __syncwarp();
  if (lane == 0) bar_arrive(&s_stg[k]);
  bar_wait(&s_stg[k], phase);
  if (t.type == TASK_Y_DENSE) {
    for (int it = 0; it < t.nterm; ++it)
      if (sl.src[2 * it + 1])
        for (int c = lane; c < m; c += 32)
          sl.vec[2 * it * m + c] = cadd(sl.vec[2 * it * m + c], sl.vec[(2 * it + 1) * m + c]);
  }
}

// all 32 lanes: poll the task's dependency counters (in parallel) until every
// producer group it reads has finished
__device__ __forceinline__ void wait_deps(const ExecArgs& a, const DevTask& t, const Slot& sl, int lane) {
  const DevWait* w = sl.waits();
  const int nw = t.nwait;
  for (int i = lane; i < nw; i += 32) CHK(w[i].ctr >= 0 && w[i].ctr < a.n_counters, CHK_COUNTER, t.q, w[i].ctr);
  SPIN_DECL;
  bool ok = true;
  for (int i = lane; i < nw; i += 32)
    if (ld_acquire(a.ctr + w[i].ctr) < w[i].val) ok = false;
  ok = __all_sync(0xffffffffu, ok);
  while (!ok) {
    SPIN_CHECK(t.q);
    if (a.poll_ns > 0) __nanosleep(a.poll_ns);
    ok = true;
    for (int i = lane; i < nw; i += 32)
      if (ld_acquire(a.ctr + w[i].ctr) < w[i].val) ok = false;
    ok = __all_sync(0xffffffffu, ok);
  }
}

// lane 0: the task's metadata blob into slot k (one bulk copy); all lanes
// wait for it (phase j of the slot's metadata barrier)
__device__ __forceinline__ void fetch_blob(const ExecArgs& a, const Slot& sl, int k, int q, int j,
                                           int lane) {
  if (lane == 0) {
    trace_mark(a, q, 0);
    const int64_t o0 = __ldg(a.blob_off + q), o1 = __ldg(a.blob_off + q + 1);
    const uint32_t bytes = (uint32_t)((o1 - o0) * 16);
    bar_expect(&s_meta[k], bytes);
    bulk_copy(sl.blob, a.blob + o0, bytes, &s_meta[k]);
  }
  bar_wait(&s_meta[k], j & 1);
}

// Producer warp k: slot k, the CTA's slot uses i = k, k + n_slots, ...
__device__ void producer(const ExecArgs& a, const Layout& L, int k) {
  const int lane = threadIdx.x & 31;
  const uint32_t ns = (uint32_t)L.n_stages;
  const Slot sl = L.slot(k);
  int n_staged = 0;  // phases of this slot's staging barrier
  for (int j = 0;; ++j) {
    const int use = L.n_slots * j + k;
    if (j > 0) {  // consumers done with the previous use: publish its outputs
      bar_wait(&s_tempty[k], (j - 1) & 1);
      if (lane == 0) {  // release: the consumers' outputs before the count
        CHK(sl.desc().signal >= 0 && sl.desc().signal < a.n_counters, CHK_COUNTER, sl.desc().q,
            sl.desc().signal);
        asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.ctr + sl.desc().signal)
                     : "memory");
      }
    }
    // one task per use, grabbed in use order (the CTA's uses run in
    // increasing queue order, which the dependency argument needs)
    int q = 0;
    if (lane == 0) {
      while (s_grab_turn != use) __nanosleep(16);
      q = atomicAdd(a.head, 1);
      s_grab_turn = use + 1;
    }
    q = __shfl_sync(0xffffffffu, q, 0);
    if (q >= a.n_tasks) {  // end: consumers stop at the first empty slot use
      if (lane == 0) {
        while (s_resv_turn != use) __nanosleep(16);
        s_resv_turn = use + 1;
        reinterpret_cast<DevTask*>(sl.blob)->type = -1;
        bar_arrive(&s_tfull[k]);
      }
      return;
    }
    fetch_blob(a, sl, k, q, j, lane);
    const DevTask& t = sl.desc();
    parse_meta(t, sl, lane);
    int issued = 0;
    uint32_t pos0 = 0;  // the use's first ring position
    if (lane == 0) {
      {
        SPIN_DECL;
        while (s_resv_turn != use) {
          SPIN_CHECK(q);
          __nanosleep(16);
        }
      }
      pos0 = s_next_pos;
      s_next_pos = pos0 + (uint32_t)t.npiece;
      __threadfence_block();
      s_resv_turn = use + 1;
      // pieces before the dependency wait, into stages already free
      while (issued < t.npiece && stage_free(L, pos0 + issued, pos0)) {
        issue_piece(a, L, sl, q, issued, pos0 + issued);
        ++issued;
      }
    }
    wait_deps(a, t, sl, lane);
    if (lane == 0) trace_mark(a, q, 1);
    __syncwarp();
    stage_vectors(a, t, sl, k, n_staged, lane);
    __syncwarp();
    if (lane == 0) {
      trace_mark(a, q, 5);
      bar_arrive(&s_tfull[k]);  // release: blob, vectors, epilogue visible to consumers
      // the rest of the task's pieces, as their stages free up
      for (; issued < t.npiece; ++issued) {
        const uint32_t pos = pos0 + issued;
        if (pos >= ns) {
          {
            SPIN_DECL;
            while (!in_window(pos, pos0, ns)) {
              SPIN_CHECK(q);
              __nanosleep(32);
            }
          }
          bar_wait(&s_empty[pos % ns], ((pos / ns) - 1) & 1);
        }
        issue_piece(a, L, sl, q, issued, pos);
      }
    }
    __syncwarp();
  }
}

// ---- consumers (warps 0-7) ---------------------------------------------------------

// profiling (trace only): consumer thread 0's cycles waiting for pieces and
// in the per-piece barrier, per task
__shared__ long long s_cyc_wait, s_cyc_sync;

// the consumers' position in the ring (every consumer thread keeps a copy)
struct Ring {
  int stage;
  uint32_t phase;
};

__device__ __forceinline__ const double2* wait_piece(const ExecArgs& a, const Layout& L,
                                                     const Ring& rg, int q, int p) {
  const long long c0 = a.trace ? clock64() : 0;
  bar_wait(&s_full[rg.stage], rg.phase);
  if (a.trace && threadIdx.x == 0) {
    s_cyc_wait += clock64() - c0;
    if (p < 8) trace_mark(a, q, 6 + p);
  }
  return L.stage(rg.stage);
}

// each consumer warp releases the stage on its own (the stage's empty
// barrier counts the 16 warps): no CTA-wide barrier per piece
__device__ __forceinline__ void release_piece(const Layout& L, Ring& rg) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) bar_arrive(&s_empty[rg.stage]);
  if (++rg.stage == L.n_stages) {
    rg.stage = 0;
    rg.phase ^= 1u;
  }
}

// T_PLR: t = scale * Vt (x_a [+ x_b]).  Each Vt row is reduced by 32, 16 or
// 8 lanes by its own length (t_lane_class); a piece's rows come in class
// order, so they tile the consumer threads in aligned units of 8 lanes: a
// 32-lane row is one warp, a 16-lane row half of one.  Lane j sums columns
// j, j + 2L, ... and j + L, j + 3L, ... into two accumulators, added, then an
// xor tree inside the row's lanes.  The summation order depends only on the
// row's length, not on how rows were packed into pieces.
__device__ __forceinline__ void run_t_plr(const ExecArgs& a, const DevTask& t, const Slot& sl,
                                          const Layout& L, Ring& rg, int q) {
  double2* T = s_slot[SLOT_T];
  const double2 sc = sl.coef[0];
  const DevItem* items = sl.items();
  if (sl.src[1]) {  // merged term: the staged slices become x_a + x_b (all consumer threads)
    const int n = t.c1 - t.c0;
    for (int c = threadIdx.x; c < n; c += CONSUMERS) sl.vec[c] = cadd(sl.vec[c], sl.vec[n + c]);
    consumer_sync();
  }
  for (int p = 0; p < t.npiece; ++p) {
    const DevPiece& pc = sl.pieces()[p];
    const int n32 = pc.e0 & 1023, n16 = (pc.e0 >> 10) & 1023, n8 = (pc.e0 >> 20) & 1023;
    const int u32 = 4 * n32, u16 = u32 + 2 * n16, units = u16 + n8;
    const double2* buf = wait_piece(a, L, rg, q, p);
    for (int u0 = 0; u0 < units; u0 += CONSUMERS / 8) {
      const int u = u0 + (int)(threadIdx.x >> 3);
      int row, lanes, lane;
      if (u < u32) {
        row = u >> 2, lanes = 32, lane = threadIdx.x & 31;
      } else if (u < u16) {
        row = n32 + ((u - u32) >> 1), lanes = 16, lane = threadIdx.x & 15;
      } else {
        row = n32 + n16 + (u - u16), lanes = 8, lane = threadIdx.x & 7;
      }
      double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
      DevItem it{};
      if (u < units) {
        it = items[pc.f0 + row];
        CHK(it.poff + it.n <= a.half_elems && it.lo + it.n <= a.src_cap &&
                t.tbase + it.hi < a.t_elems, CHK_ITEM_RANGE, q, it.poff);
        const double2* V = buf + it.poff;
        const double2* x = sl.vec + it.lo;
        int c = lane;
        for (; c + lanes < it.n; c += 2 * lanes) {
          const double2 v0 = V[c], x0 = x[c], v1 = V[c + lanes], x1 = x[c + lanes];
          acc = cfma(v0, x0, acc);
          acc2 = cfma(v1, x1, acc2);
        }
        if (c < it.n) acc = cfma(V[c], x[c], acc);
        acc = cadd(acc, acc2);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double vx = __shfl_xor_sync(0xffffffffu, acc.x, o);
        const double vy = __shfl_xor_sync(0xffffffffu, acc.y, o);
        if (o < lanes) {
          acc.x += vx;
          acc.y += vy;
        }
      }
      if (u < units && lane == 0) st_cg(T + t.tbase + it.hi, cmul(sc, acc));
    }
    release_piece(L, rg);
  }
}

// init + eyes + rhs of one output row (fixed order), from the staged rows
__device__ __forceinline__ double2 epilogue_row(const DevTask& t, const Slot& sl, int row) {
  double2 v = make_double2(0.0, 0.0);
  int k = 0;
  if (t.has_init) v = sl.epi[k++ * EXEC_EPI + row];
  for (int e = 0; e < t.neye; ++e, ++k) v = cfma(sl.coef[EXEC_TERMS + e], sl.epi[k * EXEC_EPI + row], v);
  if (t.has_rhs) {
    const double2 r = sl.epi[k * EXEC_EPI + row];
    v.x = fma(t.rhs_coef, r.x, v.x);
    v.y = fma(t.rhs_coef, r.y, v.y);
  }
  return v;
}

// Y_PLR: one PLR_TILE-row tile; thread = (row r, column group g); columns
// f = g (mod 32) ascending, two per iteration into two accumulators; the
// groups' sums per row are added in a fixed order.
__device__ __forceinline__ void run_y_plr(const ExecArgs& a, const DevTask& t, const Slot& sl,
                                          const Layout& L, Ring& rg, int q) {
  constexpr int G = CONSUMERS / PLR_TILE;
  const int r = threadIdx.x % PLR_TILE, g = threadIdx.x / PLR_TILE;
  // a column's item: offset in its stage | first tile row << 16 | end row << 20
  const uint32_t* items = reinterpret_cast<const uint32_t*>(sl.blob + t.item0);
  if (t.nsrun > 0) {
    // dense-leaf columns: the staged source values become scale * (x_a + x_b)
    // (by all consumer threads: a dense kernel's task stages ~1,000 of them,
    // too many for the producer warp's serial pass on the dependency path)
    const DevSrcRun* sr = sl.sruns();
    for (int i = 0; i < t.nsrun; ++i) {
      const DevSrcRun r = sr[i];
      const double2 sc = sl.coef[r.term];
      const bool two = sl.src[2 * r.term + 1] != nullptr;
      for (int c = threadIdx.x; c < r.n; c += CONSUMERS) {
        double2 v = sl.vec[r.f + c];
        if (two) v = cadd(v, sl.vec[t.nitem + r.b_off + c]);
        sl.vec[r.f + c] = cmul(sc, v);
      }
    }
    consumer_sync();
  }
  double2 acc = make_double2(0.0, 0.0);
  double2 acc2 = make_double2(0.0, 0.0);
  for (int p = 0; p < t.npiece; ++p) {
    const DevPiece& pc = sl.pieces()[p];
    const double2* buf = wait_piece(a, L, rg, q, p);
    int f = pc.f0 + ((g - pc.f0) % G + G) % G;
    for (; f + G < pc.f1; f += 2 * G) {
      const uint32_t w0 = items[f], w1 = items[f + G];
      const int p0 = (int)(w0 & 0xFFFFu), lo0 = (int)((w0 >> 16) & 15u), hi0 = (int)((w0 >> 20) & 31u);
      const int p1 = (int)(w1 & 0xFFFFu), lo1 = (int)((w1 >> 16) & 15u), hi1 = (int)((w1 >> 20) & 31u);
      CHK(p0 + (hi0 - lo0) <= a.half_elems && p1 + (hi1 - lo1) <= a.half_elems &&
              hi0 <= PLR_TILE && hi1 <= PLR_TILE, CHK_ITEM_RANGE, q, f);
      const double2 t0 = sl.vec[f], t1 = sl.vec[f + G];
      const double2 u0 = r >= lo0 && r < hi0 ? buf[p0 + (r - lo0)] : make_double2(0.0, 0.0);
      const double2 u1 = r >= lo1 && r < hi1 ? buf[p1 + (r - lo1)] : make_double2(0.0, 0.0);
      acc = cfma(u0, t0, acc);
      acc2 = cfma(u1, t1, acc2);
    }
    if (f < pc.f1) {
      const uint32_t w = items[f];
      const int po = (int)(w & 0xFFFFu), lo = (int)((w >> 16) & 15u), hi = (int)((w >> 20) & 31u);
      if (r >= lo && r < hi) acc = cfma(buf[po + (r - lo)], sl.vec[f], acc);
    }
    release_piece(L, rg);
  }
  // the two column groups of a warp (lanes r and r + 16) first, then the 16
  // warp sums in four interleaved chains
  double2 v = cadd(acc, acc2);
  v.x += __shfl_xor_sync(0xffffffffu, v.x, 16);
  v.y += __shfl_xor_sync(0xffffffffu, v.y, 16);
  double2* part = L.part();
  if ((threadIdx.x & 31) < PLR_TILE) part[(threadIdx.x >> 5) * PLR_TILE + r] = v;
  consumer_sync();
  if ((int)threadIdx.x < t.r1 - t.r0) {
    double2 s4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) s4[i] = part[i * PLR_TILE + threadIdx.x];
#pragma unroll
    for (int i = 4; i < CWARPS; ++i) s4[i & 3] = cadd(s4[i & 3], part[i * PLR_TILE + threadIdx.x]);
    const double2 sum = cadd(cadd(s4[0], s4[1]), cadd(s4[2], s4[3]));
    st_cg(vptr_w(t.out) + t.r0 + threadIdx.x, cadd(epilogue_row(t, sl, threadIdx.x), sum));
  }
}

// Y_DENSE: rows [r0, r1) (<= 4); piece p = rows of term p's kernel; columns
// split over the warps, per-warp scaled partials summed in warp order.
__device__ __forceinline__ void run_y_dense(const ExecArgs& a, const DevTask& t, const Slot& sl,
                                            const Layout& L, Ring& rg, int q) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = a.m;
  const int nrows = t.r1 - t.r0;
  double2* part = L.part();
  if (lane < DENSE_RT_MAX) part[warp * DENSE_RT_MAX + lane] = make_double2(0.0, 0.0);
  for (int it = 0; it < t.nterm; ++it) {
    const double2* K = wait_piece(a, L, rg, q, it);
    const double2* x = sl.vec + 2 * it * m;
    double2 d[DENSE_RT_MAX];
#pragma unroll
    for (int i = 0; i < DENSE_RT_MAX; ++i) d[i] = make_double2(0.0, 0.0);
    for (int c = 32 * warp + lane; c < m; c += CONSUMERS) {
      const double2 sv = x[c];
#pragma unroll
      for (int i = 0; i < DENSE_RT_MAX; ++i)
        if (i < nrows) d[i] = cfma(K[i * m + c], sv, d[i]);
    }
    const double2 sc = sl.coef[it];
#pragma unroll
    for (int i = 0; i < DENSE_RT_MAX; ++i) {
      const double2 rr = warp_sum(d[i]);
      if (lane == i && i < nrows)
        part[warp * DENSE_RT_MAX + i] = cfma(sc, rr, part[warp * DENSE_RT_MAX + i]);
    }
    release_piece(L, rg);
  }
  consumer_sync();
  if ((int)threadIdx.x < nrows) {
    double2 v = epilogue_row(t, sl, threadIdx.x);
    for (int w = 0; w < CWARPS; ++w) v = cadd(v, part[w * DENSE_RT_MAX + threadIdx.x]);
    st_cg(vptr_w(t.out) + t.r0 + threadIdx.x, v);
  }
}

__device__ void consumer(const ExecArgs& a, const Layout& L) {
  Ring rg{0, 0u};  // pieces consumed
  for (int use = 0;; ++use) {
    const int k = use % L.n_slots;
    const Slot sl = L.slot(k);
    bar_wait(&s_tfull[k], (use / L.n_slots) & 1);  // acquire the producer's staging
    const DevTask& t = sl.desc();
    if (t.type < 0) return;
    const int q = t.q;
    if (threadIdx.x == 0) trace_mark(a, q, 4);
    if (t.type == TASK_T_PLR)
      run_t_plr(a, t, sl, L, rg, q);
    else if (t.type == TASK_Y_PLR)
      run_y_plr(a, t, sl, L, rg, q);
    else
      run_y_dense(a, t, sl, L, rg, q);
    consumer_sync();
    if (threadIdx.x == 0) {  // the slot's producer warp publishes the outputs
      s_consumed = s_consumed + (uint32_t)t.npiece;  // every warp released the task's stages
      __threadfence_block();
      trace_mark(a, q, 2);
      trace_mark(a, q, 3);
      if (a.trace) {
        a.trace[EXEC_TRACE * (size_t)q + 22] = s_cyc_wait;
        a.trace[EXEC_TRACE * (size_t)q + 23] = s_cyc_sync;
        s_cyc_wait = s_cyc_sync = 0;
      }
      bar_arrive(&s_tempty[k]);
    }
  }
}

}  // namespace

__global__ void __launch_bounds__(EXEC_THREADS, 512 / EXEC_CONSUMERS) pt_exec_kernel(ExecArgs a) {
  extern __shared__ __align__(128) double2 smem[];
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
#if PT_CHECK
    s_errp = a.err;
#endif
    s_cyc_wait = s_cyc_sync = 0;
    s_resv_turn = 0;
    s_grab_turn = 0;
    s_next_pos = 0;
    s_consumed = 0;
    for (int i = 0; i < a.n_stages; ++i) {
      bar_init(&s_full[i], 1);
      bar_init(&s_empty[i], EXEC_CONSUMERS / 32);
    }
    for (int i = 0; i < EXEC_TSLOTS; ++i) {
      bar_init(&s_tfull[i], 1);
      bar_init(&s_tempty[i], 1);
      bar_init(&s_meta[i], 1);
      bar_init(&s_stg[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const Layout L = carve(smem, a);
  if (threadIdx.x >= CONSUMERS) {
    const int k = (threadIdx.x - CONSUMERS) >> 5;
    if (k < L.n_slots) producer(a, L, k);  // unused task slots: their warps wait below
  } else {
    consumer(a, L);
  }
  // Counters reset themselves: the last CTA out zeroes the program's
  // counters, the queue heads and the exit ticket, so the next launch needs
  // no memset node (a memset between two kernels cost ~11 us of launch gap
  // per GMRES iteration).  Every CTA's polls and signals are done here.
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(a.head + 1, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    const int n = (int)(a.head - a.ctr) + 3;
    for (int i = threadIdx.x; i < n; i += blockDim.x) a.ctr[i] = 0;
  }
}

}  // namespace pt
