// Device-side helpers shared by the executor and the GMRES kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "pt_types.h"

namespace pt {

// executor CTA (one per SM): 16 consumer warps + 3 producer warps (one per
// task slot)
#ifndef PT_EXEC_CONSUMERS
#define PT_EXEC_CONSUMERS 512
#endif
constexpr int EXEC_CONSUMERS = PT_EXEC_CONSUMERS;  // 512: one CTA per SM; 256: two
constexpr int EXEC_PRODUCERS = 3;  // = task slots
constexpr int EXEC_THREADS = EXEC_CONSUMERS + 32 * EXEC_PRODUCERS;
constexpr int EXEC_WARPS = EXEC_CONSUMERS / 32;
constexpr int EXEC_MAX_STAGES = 8;  // operator piece ring (TMA bulk copies); the
                                    // handle picks 2..8 stages from its smem budget
constexpr int EXEC_TSLOTS = EXEC_PRODUCERS;  // task slots (metadata blob, staged vectors)
constexpr int EXEC_PART = 256;      // consumer partial sums (complex), per CTA
constexpr int EXEC_EPI = 16;        // epilogue rows per task slot (>= PLR_TILE, DENSE_RT_MAX)
constexpr int EXEC_EPI_SRC = 6;     // epilogue source rows: init, eyes (<= 4), rhs
constexpr int EXEC_TERMS = 16;      // term scales per task slot
constexpr int EXEC_EYES = EXEC_EPI_SRC - 2;
constexpr int EXEC_TRACE = 24;      // u64 trace words per task (pt_trace_program)
constexpr int EXEC_PIECES = 48;     // operator pieces of one task (descriptors in the slot)
constexpr int EXEC_SRCS = 2 * EXEC_TERMS + EXEC_EPI_SRC;  // vector pointers of one task
constexpr int EXEC_WAITS = 64;      // dependency counters of one task (polled by 32 lanes)
constexpr int DENSE_RT_MAX = 4;   // max rows of a Y_DENSE task (split-K over warps)
constexpr int DENSE_ROWS_PER_TASK = 4;

__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// acc + a*b
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
// acc + conj(a)*b
__device__ __forceinline__ double2 cfma_conj(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}

// immutable operator data: read-only path, no L1 allocation (streamed once)
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}
// vectors produced inside the launch by other CTAs: L2 only (L1 is not
// coherent across SMs)
__device__ __forceinline__ double2 ld_cg(const double2* p) { return __ldcg(p); }
__device__ __forceinline__ void st_cg(double2* p, double2 v) { __stcg(p, v); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// Checked build (-DPT_CHECK=1, libpt_b200_check.so; PT_LIBRARY selects it):
// the executor asserts its index and capacity invariants and bounds every
// spin loop; a violation records (code, task, value) in ExecArgs::err and
// traps, so the launch fails instead of corrupting memory or hanging.
// compute-sanitizer is not available on the GPU pool; this is its stand-in.
#ifndef PT_CHECK
#define PT_CHECK 0
#endif
enum CheckCode : int {
  CHK_PIECE_SIZE = 1,    // operator piece larger than a ring stage
  CHK_PIECE_RANGE = 2,   // operator piece outside the operator pool
  CHK_STAGE_VEC = 3,     // staged vectors beyond the slot's vector area
  CHK_ITEM_RANGE = 4,    // an item addresses outside its ring stage
  CHK_COUNTER = 5,       // counter index outside the program's counters
  CHK_WINDOW = 6,        // ring parity window invariant broken
  CHK_HANG = 7,          // a spin loop ran longer than the watchdog
  CHK_EPI_ROWS = 8,      // more output rows than the epilogue staging holds
  CHK_SLOT_T = 9,        // t-buffer index outside SLOT_T
};

struct ExecArgs {
  const DevTask* tasks;
  const DevTerm* terms;
  const DevEye* eyes;
  const DevWait* waits;
  int* ctr;   // counters; ctr[n_counters] is the queue head
  int* head;
  double2* slot[N_SLOTS];
  const double2* dense;
  const double2* fac;
  const DevLeaf* leaves;
  const DevSlot* slots;
  const DevKernelPLR* kplr;
  const int32_t* tile_ptr;
  const DevTileEntry* tile_ent;
  const DevTileEntry* ents;  // program's Y_PLR task entries
  const DevPiece* pieces;    // program's staged operator ranges
  const DevItem* items;      // program's per-column / per-slot task metadata
  // per-task metadata blobs in queue order (see pt_api.cu build_blobs): task q
  // is blob[blob_off[q] .. blob_off[q+1]) in 16-byte units
  const int4* blob;
  const int64_t* blob_off;
  int64_t half_elems;        // complex capacity of one ring stage
  int64_t src_cap;           // complex capacity of a task slot's vector staging area
  int64_t blob_cap;          // bytes of a task slot's blob area
  int64_t slot_bytes;        // bytes of one task slot
  int32_t n_stages;          // ring stages (<= EXEC_MAX_STAGES)
  int32_t n_slots;           // task slots in use (2..EXEC_TSLOTS)
  int32_t poll_ns;           // back-off between dependency polls (0: spin)
  const int* stop;  // GMRES status stop flag: the whole launch is skipped once set
  // iteration-relative basis addressing (GMRES loop inside a graph):
  // if iter != nullptr, SLOT_IN = vbase + (*iter) * vstride, SLOT_OUT = SLOT_IN + vstride
  const int* iter;
  double2* vbase;
  int64_t vstride;
  unsigned long long* trace;  // optional per-task timeline (debug/profiling)
  int n_tasks;
  int m;
  int n_counters;
  int64_t fac_elems, dense_elems, t_elems;  // pool and SLOT_T sizes (checked build)
  long long* err;  // checked build: {code, task, value}
};

// TMA bulk prefetch of a contiguous range into L2 (no smem, no completion)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  const char* c = (const char*)p;
  while (bytes > 0) {
    const uint32_t n = bytes > 32768u ? 32768u : bytes;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(c), "r"(n) : "memory");
    c += n;
    bytes -= n;
  }
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__global__ void pt_exec_kernel(ExecArgs a);

}  // namespace pt
