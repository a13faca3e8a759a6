// C ABI (include/pt_b200.h): upload, program cache, launches, GMRES driver.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "pt_b200.h"
#include "pt_batch.cuh"
#include "pt_device.cuh"
#include "pt_gmres.cuh"
#include "pt_plan.h"

namespace pt {
static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace pt

using namespace pt;

namespace {

thread_local std::string g_err;

// checked build: the executor's {code, task, value} record of the last
// failed invariant (mapped host memory, readable after the launch traps)
std::atomic<long long*> g_check_rec{nullptr};

int fail(int code, const std::string& msg) {
  g_err = msg;
  long long* r = g_check_rec.load();
  if (r && r[0] != 0)
    g_err += " [executor check " + std::to_string(r[0]) + " at task " + std::to_string(r[1]) +
             ", value " + std::to_string(r[2]) + "]";
  return code;
}

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      return fail(PT_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));          \
  } while (0)

template <class T>
int upload(T** dst, const std::vector<T>& v) {
  *dst = nullptr;
  if (v.empty()) return 0;
  CK(cudaMalloc((void**)dst, v.size() * sizeof(T)));
  CK(cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return 0;
}

struct DevProgram {
  Program host;
  DevTask* tasks = nullptr;
  DevTerm* terms = nullptr;
  DevEye* eyes = nullptr;
  DevWait* waits = nullptr;
  DevTileEntry* ents = nullptr;
  DevPiece* pieces = nullptr;
  DevItem* items = nullptr;
  bool fused = false;          // planned and launched with the handle's fused geometry
  int4* blob = nullptr;        // per-task metadata blobs (queue order)
  int64_t* blob_off = nullptr;  // task q: blob[blob_off[q] .. blob_off[q + 1])
  ~DevProgram() {
    cudaFree(blob);
    cudaFree(blob_off);
    cudaFree(ents);
    cudaFree(pieces);
    cudaFree(items);
    cudaFree(tasks);
    cudaFree(terms);
    cudaFree(eyes);
    cudaFree(waits);
  }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

struct pt_gmres_ws {
  int device = 0;
  GmresDev d{};
  DevStatus* st_host = nullptr;  // pinned ring of 2 status snapshots
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~pt_gmres_ws() {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    cudaFree(d.ticket);
    cudaFree(d.nonfinite);
    cudaFree(d.V);
    cudaFree(d.P);
    cudaFree(d.h1);
    cudaFree(d.h2);
    cudaFree(d.hn2);
    cudaFree(d.R);
    cudaFree(d.Hraw);
    cudaFree(d.g);
    cudaFree(d.cs);
    cudaFree(d.sn);
    cudaFree(d.hist);
    cudaFree(d.y);
    cudaFree(d.st);
    cudaFreeHost(st_host);
  }
};

struct pt_handle {
  int device = 0;
  bool host_only = false;  // PT_DEVICE_HOST: plan tables only
  bool dense_leaves = true;  // store factor-heavy PLR leaves as U.Vt (PT_DENSE_LEAVES=0: off)
  Operator op;
  std::string sweep_err;
  PlanParams pp;
  double2* dense = nullptr;
  double2* fac = nullptr;
  DevLeaf* leaves = nullptr;
  DevSlot* slots = nullptr;
  DevKernelPLR* kplr = nullptr;
  int32_t* tile_ptr = nullptr;
  DevTileEntry* tile_ent = nullptr;
  std::map<std::string, std::unique_ptr<DevProgram>> progs;
  double2* slot_buf[N_SLOTS] = {nullptr};
  int64_t slot_cap[N_SLOTS] = {0};
  int* ctr = nullptr;
  int ctr_cap = 0;
  int grid = 0;
  size_t smem = 0;
  int64_t src_cap = 0;     // complex elements of a task slot's vector staging
  int64_t item_cap = 0;    // items of a task slot
  int64_t blob_cap = 0;    // bytes of a task slot's metadata blob area
  int64_t run_cap = 0;     // t-value runs of a task (PLR)
  int64_t srun_cap = 0;    // dense-leaf source runs of a task (PLR)
  int64_t slot_bytes = 0;  // bytes of one task slot
  int n_stages = 4;        // operator ring stages
  int n_slots = EXEC_TSLOTS;  // task slots in use per CTA
  int piece_cap = EXEC_PIECES;  // operator pieces of one task the slot's blob area holds
  // The executor geometry above (task-slot capacities, ring, plan parameters)
  // is the default one: programs A, M, S.  The fused A -> M iteration has its
  // own (PLR operators): its A-apply part is planned as short background
  // tasks, which need smaller task slots and leave larger ring stages.
  struct ExecGeom {
    int64_t src_cap, item_cap, blob_cap, run_cap, srun_cap, slot_bytes;
    int n_stages, n_slots, piece_cap, grid;
    size_t smem;
    PlanParams pp;
  };
  ExecGeom fused{};
  bool has_fused = false;
  ExecGeom geom() const {
    return ExecGeom{src_cap, item_cap, blob_cap, run_cap, srun_cap, slot_bytes,
                    n_stages, n_slots, piece_cap, grid, smem, pp};
  }
  void set_geom(const ExecGeom& g) {
    src_cap = g.src_cap, item_cap = g.item_cap, blob_cap = g.blob_cap, run_cap = g.run_cap;
    srun_cap = g.srun_cap, slot_bytes = g.slot_bytes, n_stages = g.n_stages, n_slots = g.n_slots;
    piece_cap = g.piece_cap, grid = g.grid, smem = g.smem, pp = g.pp;
  }
  int api_fmt = 0;         // the kernel format pt_create was given (op.fmt is the executor's storage)
  int poll_ns = 20;        // dependency-poll back-off (PT_POLL_NS)
  // Launch ordering across streams: every program launch shares the handle's
  // counters, queue heads and scratch vectors, so a launch on another stream
  // waits for the previous launch (its event) instead of racing it.
  cudaEvent_t last_ev = nullptr;
  cudaStream_t last_stream = nullptr;
  int64_t fac_elems = 0, dense_elems = 0;  // operator pool sizes (checked build)
  long long* chk_host = nullptr;           // checked build: mapped {code, task, value}
  long long* chk_dev = nullptr;
  std::unique_ptr<pt_gmres_ws> gws;
  double2* tmp = nullptr;
  double2* hb = nullptr;  // device staging for the *_host solve
  double2* hx = nullptr;
  // whole-solve CUDA graphs (conditional WHILE node), keyed by config
  struct SolveGraph {
    int n_it = 0, max_iter = 0;
    double tol = 0.0;
    int64_t k_pro = 0, k_body = 0, k_epi = 0;  // kernel nodes per part
    cudaGraphExec_t exec = nullptr;
  };
  std::vector<SolveGraph> graphs;
  cudaStream_t cap_stream = nullptr;
  double2* gb = nullptr;  // graph-owned rhs / solution buffers
  double2* gx = nullptr;
  double* hist_host = nullptr;  // pinned
  void drop_graphs() {
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    graphs.clear();
  }
  // multi-RHS path (pt_batch.cu): dense operators, BW sources per batch
  struct Batch {
    std::map<std::string, std::unique_ptr<DevProgram>> progs;
    PlanParams pp;
    int grid = 0;  // persistent CTAs of the batched executor
    int rows = BT_ROWS;  // output rows per task (8 or 16)
    int tcols = 32;      // sources per task (32: every task split in two source halves,
                         // 16 x 32 tiles -- c5 0.185 ms per source vs 0.200 at 8 x 64)
    double2* slot[N_SLOTS] = {nullptr};
    int64_t slot_cap[N_SLOTS] = {0};
    int* ctr = nullptr;
    int ctr_cap = 0;
    BGmresDev g{};
    int g_iter = 0;  // max_iter the GMRES arrays are sized for
    double2* b = nullptr;     // batched rhs / solution / scratch (N x BW)
    double2* x = nullptr;
    double2* tmp = nullptr;
    double2* cols = nullptr;  // column-major staging of the *_host calls
    DevStatus* st_host = nullptr;  // pinned: BW statuses + the control words
    double* hist_host = nullptr;   // pinned: BW x max_iter
    int* ctl_host = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    struct Graph {
      int n_it = 0, max_iter = 0, nrhs = 0;
      double tol = 0.0;
      int64_t k_pro = 0, k_body = 0, k_epi = 0;
      cudaGraphExec_t exec = nullptr;
    };
    std::vector<Graph> graphs;
    void drop_graphs() {
      for (auto& gr : graphs) cudaGraphExecDestroy(gr.exec);
      graphs.clear();
    }
    void free_gmres() {
      for (void* p : {(void*)g.V, (void*)g.P, (void*)g.h1, (void*)g.h2, (void*)g.R, (void*)g.g,
                      (void*)g.cs, (void*)g.sn, (void*)g.hist, (void*)g.y, (void*)g.inv,
                      (void*)g.st, (void*)g.ctl})
        cudaFree(p);
      g = BGmresDev{};
      cudaFreeHost(st_host);
      cudaFreeHost(hist_host);
      cudaFreeHost(ctl_host);
      st_host = nullptr;
      hist_host = nullptr;
      ctl_host = nullptr;
      g_iter = 0;
    }
    ~Batch() {
      drop_graphs();
      free_gmres();
      for (auto e : ev)
        if (e) cudaEventDestroy(e);
      progs.clear();
      for (int s = 0; s < N_SLOTS; ++s) cudaFree(slot[s]);
      cudaFree(ctr);
      cudaFree(b);
      cudaFree(x);
      cudaFree(tmp);
      cudaFree(cols);
    }
  } batch;
  // per-task timeline of one traced launch (pt_trace_program)
  unsigned long long* trace_buf = nullptr;
  // per-launch instrumentation of the executor
  bool timing = false;
  std::vector<cudaEvent_t> ev_free;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_used;
  int64_t timed_launches = 0, timed_bytes = 0;
  ~pt_handle() {
    for (auto& p : ev_used) {
      cudaEventDestroy(p.first);
      cudaEventDestroy(p.second);
    }
    for (auto e : ev_free) cudaEventDestroy(e);
    if (last_ev) cudaEventDestroy(last_ev);
    if (chk_host) {
      if (g_check_rec.load() == chk_host) g_check_rec.store(nullptr);
      cudaFreeHost(chk_host);
    }
    drop_graphs();
    if (cap_stream) cudaStreamDestroy(cap_stream);
    cudaFree(gb);
    cudaFree(gx);
    cudaFreeHost(hist_host);
    progs.clear();
    cudaFree(dense);
    cudaFree(fac);
    cudaFree(leaves);
    cudaFree(slots);
    cudaFree(kplr);
    cudaFree(tile_ptr);
    cudaFree(tile_ent);
    for (int s = 0; s < N_SLOTS; ++s) cudaFree(slot_buf[s]);
    cudaFree(ctr);
    cudaFree(tmp);
    cudaFree(hb);
    cudaFree(hx);
  }
  int64_t N() const { return op.nb * op.m; }
};

namespace {

// Device layout of the PLR factors, per kernel:
//   Vt region  -- every slot's Vt row (leaf order, rank order), contiguous,
//                 so the slots of a T task are one bulk copy;
//   U chunks   -- per PLR_TILE-row tile: for each leaf meeting the tile, for
//                 each rank column, the tile's rows of U*Sigma (column-major
//                 pieces), so the U data of one Y task term is one range.
// Bytes are the reference's factor bytes (plus 128-byte alignment pads).
int build_plr_tables(pt_handle* h, const pt_leaf* leaves, int64_t n_leaves, const double* fac,
                     int64_t n_fac) {
  Operator& op = h->op;
  const int64_t m = op.m;
  std::vector<int64_t> idx;
  for (int64_t i = 0; i < n_leaves; ++i) {
    const pt_leaf& L = leaves[i];
    if (L.kernel < 0 || L.kernel >= op.nk)
      return fail(PT_EINVAL, "PLR leaf references an unknown kernel");
    if (L.rank < 0 || L.rows < 0 || L.cols < 0 || L.row_off < 0 || L.col_off < 0 ||
        L.row_off + L.rows > m || L.col_off + L.cols > m)
      return fail(PT_EINVAL, "PLR leaf lies outside its m x m block");
    if (L.rank > 0 && (L.u_off < 0 || L.vt_off < 0 || L.u_off + L.rows * L.rank > n_fac ||
                       L.vt_off + L.rank * L.cols > n_fac))
      return fail(PT_EINVAL, "PLR leaf factors lie outside the factor array");
    idx.push_back(i);
  }
  std::stable_sort(idx.begin(), idx.end(),
                   [&](int64_t a, int64_t b) { return leaves[a].kernel < leaves[b].kernel; });
  std::vector<double2> blob;
  auto align8 = [&]() {
    while (blob.size() % 8) blob.push_back(make_double2(0.0, 0.0));
  };
  auto U = [&](const pt_leaf& L, int64_t r, int64_t c) {  // (U*Sigma)[r, c], row-major input
    const double* z = fac + 2 * (L.u_off + r * L.rank + c);
    return make_double2(z[0], z[1]);
  };
  op.kplr.assign(op.nk, DevKernelPLR{});
  op.nslot.assign(op.nk, 0);
  op.kernel_bytes.assign(op.nk, 0);
  const int64_t ntiles = (m + PLR_TILE - 1) / PLR_TILE;
  size_t pos = 0;
  for (int k = 0; k < op.nk; ++k) {
    DevKernelPLR& kp = op.kplr[k];
    kp.leaf0 = (int32_t)op.leaves.size();
    kp.slot0 = (int32_t)op.slots.size();
    std::vector<const pt_leaf*> kl;
    for (; pos < idx.size() && leaves[idx[pos]].kernel == k; ++pos) {
      const pt_leaf& L = leaves[idx[pos]];
      op.kernel_bytes[k] += 16 * L.rank * (L.rows + L.cols);  // the reference's bytes
      if (L.rank > 0) kl.push_back(&L);
    }
    // a dense kernel carried as one full leaf with Vt = I (mixed operators,
    // e.g. the dense E blocks of the extrapolation variant next to compressed
    // Green's blocks): the reference reads its m x m entries
    if (kl.size() == 1 && kl[0]->row_off == 0 && kl[0]->col_off == 0 && kl[0]->rows == m &&
        kl[0]->cols == m && kl[0]->rank == m) {
      bool eye = true;
      for (int64_t r = 0; r < m && eye; ++r)
        for (int64_t c = 0; c < m && eye; ++c) {
          const double* z = fac + 2 * (kl[0]->vt_off + r * m + c);
          eye = z[0] == (r == c ? 1.0 : 0.0) && z[1] == 0.0;
        }
      if (eye) op.kernel_bytes[k] = 16 * m * m;
    }
    // leaves whose factors outweigh their product are stored as the product
    // U.Vt (FP64, the same matrix to rounding): fewer bytes, and no T work
    auto dense_leaf = [&](const pt_leaf* L) {
      return h->dense_leaves && L->rank * (L->rows + L->cols) > L->rows * L->cols;
    };
    // slots ordered by column band: a T task's run of slots then reads a
    // narrow range of the source vector
    std::stable_sort(kl.begin(), kl.end(), [](const pt_leaf* a, const pt_leaf* b) {
      return a->col_off != b->col_off ? a->col_off < b->col_off : a->row_off < b->row_off;
    });
    // Vt region
    align8();
    int32_t slot = 0;
    for (const pt_leaf* L : kl) {
      DevLeaf dl{};
      dl.row_off = (int32_t)L->row_off;
      dl.col_off = (int32_t)L->col_off;
      dl.rows = (int32_t)L->rows;
      dl.cols = (int32_t)L->cols;
      dl.rank = (int32_t)L->rank;
      dl.slot0 = slot;
      dl.v_off = (int64_t)blob.size();
      if (dense_leaf(L)) {  // no Vt rows: the leaf's columns act as its "rank" columns
        dl.slot0 = -1;
        op.leaves.push_back(dl);
        continue;
      }
      const double* Vt = fac + 2 * L->vt_off;
      for (int64_t c = 0; c < L->rank; ++c) {
        DevSlot sl{};
        sl.v_off = (int64_t)blob.size();
        sl.col_off = dl.col_off;
        sl.cols = dl.cols;
        op.slots.push_back(sl);
        for (int64_t j = 0; j < L->cols; ++j)
          blob.push_back(make_double2(Vt[2 * (c * L->cols + j)], Vt[2 * (c * L->cols + j) + 1]));
      }
      slot += (int32_t)L->rank;
      op.leaves.push_back(dl);
    }
    kp.nleaf = (int32_t)op.leaves.size() - kp.leaf0;
    kp.nslot = slot;
    op.nslot[k] = slot;
    // tile-major U chunks
    kp.tile0 = (int32_t)op.tile_ptr.size();
    for (int64_t t = 0; t < ntiles; ++t) {
      align8();
      op.tile_ptr.push_back((int32_t)op.tile_ent.size());
      op.tile_chunk.push_back((int64_t)blob.size());
      const int64_t lo = t * PLR_TILE, hi = std::min<int64_t>(m, lo + PLR_TILE);
      for (int32_t l = 0; l < kp.nleaf; ++l) {
        const DevLeaf& dl = op.leaves[kp.leaf0 + l];
        if (!(dl.row_off < hi && dl.row_off + dl.rows > lo)) continue;
        const pt_leaf& L = *kl[l];
        const int64_t r_first = std::max<int64_t>(lo, dl.row_off);
        const int64_t r_end = std::min<int64_t>(hi, dl.row_off + dl.rows);
        DevTileEntry te{};
        te.u0 = (int64_t)blob.size();
        te.t0 = dl.slot0;
        te.stride = (int32_t)(r_end - r_first);
        te.rank = dl.rank;
        te.lo = (int16_t)(r_first - lo);
        te.hi = (int16_t)(r_end - lo);
        if (dl.slot0 < 0) {  // dense leaf: the tile's rows of U.Vt, column by column
          te.rank = dl.cols;
          te.pre = dl.col_off;
          const double* Vt = fac + 2 * L.vt_off;
          for (int64_t c = 0; c < L.cols; ++c)
            for (int64_t r = r_first; r < r_end; ++r) {
              double re = 0.0, im = 0.0;
              for (int64_t j = 0; j < L.rank; ++j) {
                const double2 u = U(L, r - dl.row_off, j);
                const double vr = Vt[2 * (j * L.cols + c)], vi = Vt[2 * (j * L.cols + c) + 1];
                re = std::fma(u.x, vr, std::fma(-u.y, vi, re));
                im = std::fma(u.x, vi, std::fma(u.y, vr, im));
              }
              blob.push_back(make_double2(re, im));
            }
        } else {
          for (int64_t c = 0; c < L.rank; ++c)
            for (int64_t r = r_first; r < r_end; ++r) blob.push_back(U(L, r - dl.row_off, c));
        }
        op.tile_ent.push_back(te);
      }
    }
    op.tile_ptr.push_back((int32_t)op.tile_ent.size());
    op.tile_chunk.push_back((int64_t)blob.size());
  }
  if (op.tile_ent.empty()) op.tile_ent.push_back(DevTileEntry{});
  if (blob.empty()) blob.push_back(make_double2(0.0, 0.0));
  if (h->host_only) return 0;
  int rc;
  if ((rc = upload(&h->fac, blob))) return rc;
  h->fac_elems = (int64_t)blob.size();
  if ((rc = upload(&h->slots, op.slots))) return rc;
  if ((rc = upload(&h->kplr, op.kplr))) return rc;
  return 0;
}

// Dense kernels for the single-source executor: the same tile-major storage
// as a PLR kernel's dense leaves (one full leaf per kernel: for each 16-row
// tile, column by column, the tile's rows), so dense operators run the
// 16-row Y_PLR tasks -- a task stages its source vectors once per 16 output
// rows, and the consumers read conflict-free 16-row columns.  The row-major
// pool stays for the batched executor.  Same bytes as the m x m kernels.
int build_dense_tiles(pt_handle* h, const double* dense) {
  Operator& op = h->op;
  const int64_t m = op.m;
  const int64_t ntiles = (m + PLR_TILE - 1) / PLR_TILE;
  std::vector<double2> blob;
  blob.reserve((size_t)op.nk * m * m + 8 * (size_t)op.nk * ntiles);
  op.kplr.assign(op.nk, DevKernelPLR{});
  op.nslot.assign(op.nk, 0);
  for (int k = 0; k < op.nk; ++k) {
    const double* K = h->host_only ? nullptr : dense + 2 * (size_t)k * m * m;
    DevKernelPLR& kp = op.kplr[k];
    kp.leaf0 = (int32_t)op.leaves.size();
    kp.slot0 = (int32_t)op.slots.size();
    kp.nleaf = 1;
    kp.nslot = 0;
    DevLeaf dl{};
    dl.rows = dl.cols = dl.rank = (int32_t)m;
    dl.slot0 = -1;
    dl.v_off = (int64_t)blob.size();
    op.leaves.push_back(dl);
    kp.tile0 = (int32_t)op.tile_ptr.size();
    for (int64_t t = 0; t < ntiles; ++t) {
      while (blob.size() % 8) blob.push_back(make_double2(0.0, 0.0));
      op.tile_ptr.push_back((int32_t)op.tile_ent.size());
      op.tile_chunk.push_back((int64_t)blob.size());
      const int64_t lo = t * PLR_TILE, hi = std::min<int64_t>(m, lo + PLR_TILE);
      DevTileEntry te{};
      te.u0 = (int64_t)blob.size();
      te.t0 = -1;
      te.stride = (int32_t)(hi - lo);
      te.rank = (int32_t)m;
      te.pre = 0;
      te.lo = 0;
      te.hi = (int16_t)(hi - lo);
      if (K) {
        for (int64_t c = 0; c < m; ++c)
          for (int64_t r = lo; r < hi; ++r)
            blob.push_back(make_double2(K[2 * (r * m + c)], K[2 * (r * m + c) + 1]));
      } else {
        blob.resize(blob.size() + (size_t)((hi - lo) * m));
      }
      op.tile_ent.push_back(te);
    }
    op.tile_ptr.push_back((int32_t)op.tile_ent.size());
    op.tile_chunk.push_back((int64_t)blob.size());
  }
  if (op.tile_ent.empty()) op.tile_ent.push_back(DevTileEntry{});
  if (blob.empty()) blob.push_back(make_double2(0.0, 0.0));
  h->fac_elems = (int64_t)blob.size();
  if (h->host_only) return 0;
  int rc;
  if ((rc = upload(&h->fac, blob))) return rc;
  if ((rc = upload(&h->kplr, op.kplr))) return rc;
  return 0;
}

int ensure_slot(pt_handle* h, int s, int64_t elems) {
  if (elems <= h->slot_cap[s]) return 0;
  CK(cudaDeviceSynchronize());
  h->drop_graphs();
  cudaFree(h->slot_buf[s]);
  h->slot_buf[s] = nullptr;
  CK(cudaMalloc(&h->slot_buf[s], (size_t)std::max<int64_t>(elems, 1) * sizeof(double2)));
  CK(cudaMemset(h->slot_buf[s], 0, (size_t)std::max<int64_t>(elems, 1) * sizeof(double2)));
  h->slot_cap[s] = elems;
  return 0;
}

// Per-task metadata blobs, in queue order, so a producer warp fetches a
// task's whole description with one bulk copy:
//   [DevTask][DevPiece x npiece][DevTerm x nterm][DevEye x neye]
//   [DevWait x nwait][DevRun x nrun][DevSrcRun x nsrun][DevItem x nitem (T) | packed uint32 x nitem (Y)]
// each section 16-byte aligned.  In the blob copy of the DevTask, piece0 /
// term0 / eye0 / wait0 / run0 / srun0 / item0 are byte offsets of the sections and
// q is the queue index.
int64_t blob_bytes_max(int64_t item_cap, int64_t run_cap, int64_t srun_cap) {
  auto al = [](int64_t b) { return (b + 15) / 16 * 16; };
  return al(sizeof(DevTask)) + al(EXEC_PIECES * sizeof(DevPiece)) + al(EXEC_TERMS * sizeof(DevTerm)) +
         al(EXEC_EYES * sizeof(DevEye)) + al(EXEC_WAITS * sizeof(DevWait)) +
         al(run_cap * (int64_t)sizeof(DevRun)) + al(srun_cap * (int64_t)sizeof(DevSrcRun)) +
         al(item_cap * (int64_t)sizeof(DevItem));
}

void build_blobs(const Program& pg, std::vector<int4>& blob, std::vector<int64_t>& off,
                 int64_t* max_bytes) {
  std::vector<char> b;
  off.assign(pg.tasks.size() + 1, 0);
  *max_bytes = 0;
  auto put = [&](const void* p, size_t n) {
    const int32_t at = (int32_t)b.size();
    b.insert(b.end(), (const char*)p, (const char*)p + n);
    while (b.size() % 16) b.push_back(0);
    return at;
  };
  for (size_t q = 0; q < pg.tasks.size(); ++q) {
    const DevTask& t = pg.tasks[q];
    b.clear();
    DevTask d = t;
    put(&d, sizeof(DevTask));
    d.piece0 = put(pg.pieces.data() + t.piece0, (size_t)t.npiece * sizeof(DevPiece));
    d.term0 = put(pg.terms.data() + t.term0, (size_t)t.nterm * sizeof(DevTerm));
    d.eye0 = put(pg.eyes.data() + t.eye0, (size_t)t.neye * sizeof(DevEye));
    d.wait0 = put(pg.waits.data() + t.wait0, (size_t)t.nwait * sizeof(DevWait));
    d.run0 = put(pg.runs.data() + t.run0, (size_t)t.nrun * sizeof(DevRun));
    d.srun0 = put(pg.sruns.data() + t.srun0, (size_t)t.nsrun * sizeof(DevSrcRun));
    if (t.type == TASK_Y_PLR) {
      // a Y column's item in 4 bytes: offset in its stage | first tile row << 16 | end row << 20
      std::vector<uint32_t> packed((size_t)t.nitem);
      for (int32_t i = 0; i < t.nitem; ++i) {
        const DevItem& it = pg.items[(size_t)t.item0 + i];
        packed[i] = (uint32_t)it.poff | ((uint32_t)it.lo << 16) | ((uint32_t)it.hi << 20);
      }
      d.item0 = put(packed.data(), packed.size() * sizeof(uint32_t));
    } else {
      d.item0 = put(pg.items.data() + t.item0, (size_t)t.nitem * sizeof(DevItem));
    }
    d.q = (int32_t)q;
    std::memcpy(b.data(), &d, sizeof(DevTask));
    *max_bytes = std::max<int64_t>(*max_bytes, (int64_t)b.size());
    const size_t at = blob.size();
    blob.resize(at + b.size() / 16);
    std::memcpy(blob.data() + at, b.data(), b.size());
    off[q + 1] = (int64_t)blob.size();
  }
}

// Every task of a program fits the executor's task slot (the handle sized the
// slots from the operator; a program that does not fit is rejected).
int check_slots(const pt_handle* h, const Program& pg) {
  for (const DevTask& t : pg.tasks) {  // what one task slot stages
    int64_t vec = 0;
    if (t.type == TASK_T_PLR) vec = 2 * (t.c1 - t.c0);  // both sources of a merged term
    if (t.type == TASK_Y_PLR) vec = t.nitem + t.ndense2;
    if (t.type == TASK_Y_DENSE) vec = 2 * (int64_t)t.nterm * h->op.m;
    const int rows = t.type == TASK_Y_DENSE ? DENSE_RT_MAX : EXEC_EPI;
    if (vec > h->src_cap || t.nitem > h->item_cap || t.nterm > EXEC_TERMS ||
        t.neye > EXEC_EYES || t.npiece > h->piece_cap ||
        t.nwait > EXEC_WAITS ||
        t.nrun > h->run_cap || t.nsrun > h->srun_cap ||
        (t.type != TASK_T_PLR && t.r1 - t.r0 > rows))
      return fail(PT_EINVAL, "a task stages more than the executor's task slot holds");
  }
  return 0;
}

// The fused A -> M iteration's executor geometry while it is in scope.
// Beside a sweep chain the A-apply is background work, and a chain task that
// becomes ready waits for the background task its CTA's consumers are in:
// short background tasks (block rows as two-term partial sums, T tasks of two
// ring pieces) cost the A-apply alone ~20%, but they need smaller task slots,
// which leaves larger ring stages, and shorten every sweep level (c3 GMRES
// 17.46 -> 16.96 ms).  The stand-alone programs keep the default geometry.
struct FusedGeom {
  pt_handle* h;
  pt_handle::ExecGeom saved;
  bool on;
  FusedGeom(pt_handle* h_, bool use) : h(h_), on(use && h_->has_fused) {
    if (on) {
      saved = h->geom();
      h->set_geom(h->fused);
    }
  }
  ~FusedGeom() {
    if (on) h->set_geom(saved);
  }
};

int get_program(pt_handle* h, const std::string& kind, int n_it, DevProgram** out) {
  const std::string key = kind + std::to_string(n_it);
  auto it = h->progs.find(key);
  if (it != h->progs.end()) {
    *out = it->second.get();
    return 0;
  }
  std::unique_ptr<DevProgram> p(new DevProgram());
  p->fused = kind == "AM" && h->has_fused;
  FusedGeom scope(h, p->fused);
  if (kind == "A")
    p->host = build_apply_A(h->op, h->pp);
  else if (kind == "M")
    p->host = build_apply_M(h->op, n_it, h->pp);
  else if (kind == "S")
    p->host = build_gs_sweep(h->op, h->pp);
  else
    p->host = build_A_then_M(h->op, n_it, h->pp);
  if (!p->host.overflow.empty()) return fail(PT_EINVAL, p->host.overflow);
  if (int rc = check_slots(h, p->host)) return rc;
  int rc;
  if ((rc = upload(&p->tasks, p->host.tasks))) return rc;
  if ((rc = upload(&p->terms, p->host.terms))) return rc;
  if ((rc = upload(&p->eyes, p->host.eyes))) return rc;
  if ((rc = upload(&p->waits, p->host.waits))) return rc;
  if ((rc = upload(&p->ents, p->host.ents))) return rc;
  if ((rc = upload(&p->pieces, p->host.pieces))) return rc;
  if ((rc = upload(&p->items, p->host.items))) return rc;
  {
    std::vector<int4> blob;
    std::vector<int64_t> off;
    int64_t mx = 0;
    build_blobs(p->host, blob, off, &mx);
    if (mx > h->blob_cap) return fail(PT_EINVAL, "a task's metadata exceeds the executor's task slot");
    if ((rc = upload(&p->blob, blob))) return rc;
    if ((rc = upload(&p->blob_off, off))) return rc;
  }
  for (int s : {SLOT_Y, SLOT_U1, SLOT_U2, SLOT_PRE, SLOT_T})
    if ((rc = ensure_slot(h, s, p->host.slot_elems[s]))) return rc;
  // counters + queue head + exit ticket + chain queue head; zero between
  // launches (the executor's last CTA resets them)
  if (p->host.n_counters + 3 > h->ctr_cap) {
    CK(cudaDeviceSynchronize());
    h->drop_graphs();
    cudaFree(h->ctr);
    h->ctr_cap = p->host.n_counters + 3;
    CK(cudaMalloc(&h->ctr, h->ctr_cap * sizeof(int)));
    CK(cudaMemset(h->ctr, 0, h->ctr_cap * sizeof(int)));
    CK(cudaDeviceSynchronize());
  }
  *out = p.get();
  h->progs[key] = std::move(p);
  return 0;
}

struct IterMode {
  const int* iter = nullptr;  // device iteration counter (st->iterations)
  double2* vbase = nullptr;   // basis
  int64_t vstride = 0;
};

// before / after a launch of an executor program on stream s (see last_ev)
int order_before(pt_handle* h, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(s, &cs));
  if (cs != cudaStreamCaptureStatusNone) return 0;  // graph nodes: ordered by the graph
  if (h->last_ev && h->last_stream != s) CK(cudaStreamWaitEvent(s, h->last_ev, 0));
  return 0;
}
int order_after(pt_handle* h, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(s, &cs));
  if (cs != cudaStreamCaptureStatusNone) return 0;
  if (!h->last_ev) CK(cudaEventCreateWithFlags(&h->last_ev, cudaEventDisableTiming));
  CK(cudaEventRecord(h->last_ev, s));
  h->last_stream = s;
  return 0;
}

int run_program(pt_handle* h, DevProgram* p, const double2* in, double2* out, const double2* aux,
                cudaStream_t s, const int* stop = nullptr, IterMode im = IterMode()) {
  if (p->host.tasks.empty()) return 0;
  FusedGeom scope(h, p->fused);
  ExecArgs a{};
  a.tasks = p->tasks;
  a.terms = p->terms;
  a.eyes = p->eyes;
  a.waits = p->waits;
  a.ctr = h->ctr;
  a.head = h->ctr + p->host.n_counters;
  for (int i = 0; i < N_SLOTS; ++i) a.slot[i] = h->slot_buf[i];
  a.slot[SLOT_IN] = const_cast<double2*>(in);
  a.slot[SLOT_OUT] = out;
  a.slot[SLOT_AUX] = const_cast<double2*>(aux);
  a.dense = h->dense;
  a.fac = h->fac;
  a.leaves = h->leaves;
  a.slots = h->slots;
  a.kplr = h->kplr;
  a.tile_ptr = h->tile_ptr;
  a.tile_ent = h->tile_ent;
  a.ents = p->ents;
  a.pieces = p->pieces;
  a.items = p->items;
  a.blob = p->blob;
  a.blob_off = p->blob_off;
  a.blob_cap = h->blob_cap;
  a.half_elems = h->pp.half_elems;
  a.src_cap = h->src_cap;
  a.slot_bytes = h->slot_bytes;
  a.n_stages = h->n_stages;
  a.n_slots = h->n_slots;
  a.poll_ns = h->poll_ns;
  a.n_tasks = (int)p->host.tasks.size();
  a.m = (int)h->op.m;
  a.n_counters = p->host.n_counters;
  a.fac_elems = h->fac_elems;
  a.dense_elems = h->dense_elems;
  a.t_elems = h->slot_cap[SLOT_T];
  if (h->chk_host) {  // checked build (allocated at pt_create)
    g_check_rec.store(h->chk_host);
    a.err = h->chk_dev;
  }
  a.stop = stop;
  a.iter = im.iter;
  a.vbase = im.vbase;
  a.vstride = im.vstride;
  a.trace = h->trace_buf;
  count_launch();
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (h->timing) {
    for (cudaEvent_t* e : {&e0, &e1}) {
      if (h->ev_free.empty()) {
        CK(cudaEventCreate(e));
      } else {
        *e = h->ev_free.back();
        h->ev_free.pop_back();
      }
    }
    CK(cudaEventRecord(e0, s));
  }
  // cooperative: every CTA resident (counter waits cannot deadlock); launched
  // through cudaLaunchKernelEx so it can also be captured into a graph
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(h->grid);
  cfg.blockDim = dim3(EXEC_THREADS);
  cfg.dynamicSmemBytes = h->smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int orc = order_before(h, s);
  if (orc) return orc;
  CK(cudaLaunchKernelEx(&cfg, pt_exec_kernel, a));
  if ((orc = order_after(h, s))) return orc;
  if (h->timing) {
    CK(cudaEventRecord(e1, s));
    h->ev_used.emplace_back(e0, e1);
    h->timed_launches += 1;
    h->timed_bytes += p->host.algo_bytes;
  }
  return 0;
}

int ws_alloc(pt_gmres_ws* w, int64_t n, int max_iter) {
  GmresDev& d = w->d;
  d.n = n;
  d.max_iter = max_iter;
  d.ldp = max_iter + 2;
  const size_t ldr = (size_t)max_iter + 1;
  CK(cudaMalloc(&d.V, (size_t)n * ldr * sizeof(double2)));
  CK(cudaMalloc(&d.P, 2 * (size_t)RED_BLOCKS * d.ldp * sizeof(double2)));
  CK(cudaMalloc(&d.h1, (max_iter + 2) * sizeof(double2)));
  CK(cudaMalloc(&d.h2, (max_iter + 2) * sizeof(double2)));
  CK(cudaMalloc(&d.hn2, 2 * sizeof(double2)));
  CK(cudaMalloc(&d.R, ldr * max_iter * sizeof(double2)));
  CK(cudaMalloc(&d.Hraw, ldr * max_iter * sizeof(double2)));
  CK(cudaMalloc(&d.g, ldr * sizeof(double2)));
  CK(cudaMalloc(&d.cs, max_iter * sizeof(double)));
  CK(cudaMalloc(&d.sn, max_iter * sizeof(double2)));
  CK(cudaMalloc(&d.hist, max_iter * sizeof(double)));
  CK(cudaMalloc(&d.y, ldr * sizeof(double2)));
  CK(cudaMalloc(&d.st, sizeof(DevStatus)));
  CK(cudaMalloc(&d.nonfinite, sizeof(int)));
  CK(cudaMalloc(&d.ticket, 4 * sizeof(int)));
  CK(cudaMallocHost(&w->st_host, 2 * sizeof(DevStatus)));
  CK(cudaMemset(d.st, 0, sizeof(DevStatus)));
  CK(cudaMemset(d.nonfinite, 0, sizeof(int)));
  CK(cudaMemset(d.ticket, 0, 4 * sizeof(int)));
  for (auto& e : w->ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(gm_arnoldi_setup(d, w->device));
  return 0;
}

int fetch_status(pt_gmres_ws* w, cudaStream_t s, int slot = 0) {
  CK(cudaMemcpyAsync(w->st_host + slot, w->d.st, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}

int ws_begin_impl(pt_gmres_ws* w, const double* mb, double* beta_out, cudaStream_t s,
                  bool sync) {
  GmresDev& d = w->d;
  if ((const double2*)mb != d.V)
    CK(cudaMemcpyAsync(d.V, mb, d.n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  gm_begin(d, 0, s);
  CK(cudaGetLastError());
  if (!sync) return 0;
  int rc = fetch_status(w, s);
  if (rc) return rc;
  if (beta_out) *beta_out = w->st_host->beta;
  return 0;
}

void fill_report(const DevStatus& st, pt_report* rep) {
  rep->iterations = st.iterations;
  rep->flag = st.flag;
  rep->converged = st.converged;
  rep->beta = st.beta;
  rep->nonfinite = st.nonfinite;
}

int ws_step_impl(pt_gmres_ws* w, int j, double rel_tol, int max_iter, pt_report* rep, int* stop,
                 cudaStream_t s) {
  GmresDev& d = w->d;
  if (j < 0 || j >= d.max_iter || max_iter > d.max_iter)
    return fail(PT_EINVAL, "GMRES step index outside the workspace");
  CK(gm_arnoldi_step(d, rel_tol, max_iter, 0, s));
  CK(cudaGetLastError());
  int rc = fetch_status(w, s);
  if (rc) return rc;
  const DevStatus& st = *w->st_host;
  if (st.iterations != j + 1 && !st.nonfinite && !st.stop)
    return fail(PT_EINVAL, "GMRES steps must be taken in order");
  if (st.nonfinite) {
    if (rep) rep->nonfinite = 1;
    return fail(PT_ENONFINITE, "non-finite values in preconditioned matvec at iteration " +
                                   std::to_string(j + 1));
  }
  if (rep) {
    fill_report(st, rep);
    if (rep->residual_history && st.iterations == j + 1) rep->residual_history[j] = st.rel;
  }
  *stop = st.stop;
  return 0;
}

int ensure_gws(pt_handle* h, int max_iter) {
  if (h->gws && h->gws->d.max_iter >= max_iter) return 0;
  CK(cudaDeviceSynchronize());
  h->drop_graphs();
  cudaFreeHost(h->hist_host);
  h->hist_host = nullptr;
  CK(cudaMallocHost(&h->hist_host, (size_t)max_iter * sizeof(double)));
  h->gws.reset(new pt_gmres_ws());
  h->gws->device = h->device;
  return ws_alloc(h->gws.get(), h->N(), max_iter);
}

int check_cfg(const pt_gmres_config* cfg) {
  if (!cfg) return fail(PT_EINVAL, "missing GMRES config");
  if (!(cfg->rel_tol > 0.0 && cfg->rel_tol < 1.0)) return fail(PT_EINVAL, "rel_tol must lie in (0, 1)");
  if (cfg->max_iter < 1) return fail(PT_EINVAL, "max_iter must be at least 1");
  if (cfg->n_it < 1) return fail(PT_EINVAL, "n_it must be at least 1");
  return 0;
}

}  // namespace

extern "C" {

const char* pt_last_error(void) { return g_err.c_str(); }
int32_t pt_abi_version(void) { return PT_ABI_VERSION; }
int64_t pt_launch_count(void) { return pt::g_launches.load(); }
int32_t pt_checked_build(void) { return PT_CHECK; }

// Executor geometry of a handle from its operator and the plan parameters
// already set in h->pp (max_block_terms; want_t_pieces): task-slot capacities,
// ring stages, shared memory, grid, and the remaining plan parameters.
int size_executor(pt_handle* h, bool host_only, int device, int want_t_pieces) {
  Operator& op = h->op;
  // Shared memory per CTA: [EXEC_STAGES operator ring stages][EXEC_TSLOTS task
  // slots: descriptor, items, staged vectors, epilogue rows, term scales]
  // [consumer partials].  The stages take what is left after the fixed part
  // at one CTA per SM (the loop admits more if EXEC_THREADS shrinks) for which one
  // stage still holds the largest contiguous unit a task stages (a dense
  // kernel row, a Vt row, a tile column).
  int64_t need = op.m;  // dense: one kernel row
  if (op.fmt == PT_KERNEL_PLR) {
    need = PLR_TILE;
    for (const DevSlot& sl : op.slots) need = std::max<int64_t>(need, sl.cols);
    // a Y_PLR task stages one item and one t value per rank column meeting its
    // row tile (all terms; independent of the stage size), a T_PLR task one
    // item per Vt row (<= MAX_T_SLOTS) and a source slice (<= tcols_cap)
    PlanParams probe;
    probe.half_elems = (int64_t)1 << 30;
    probe.max_block_terms = h->pp.max_block_terms;
    int64_t ycols = 0, yvec = 0;
    for (const Program& pg : {build_apply_A(op, probe), build_apply_M(op, 2, probe),
                              build_gs_sweep(op, probe)})
      for (const DevTask& t : pg.tasks)
        if (t.type == TASK_Y_PLR) {
          ycols = std::max<int64_t>(ycols, t.nitem);
          yvec = std::max<int64_t>(yvec, t.nitem + t.ndense2);
          h->run_cap = std::max<int64_t>(h->run_cap, t.nrun);
          h->srun_cap = std::max<int64_t>(h->srun_cap, t.nsrun);
        }
    int64_t widest = 0;
    for (const DevSlot& sl : op.slots) widest = std::max<int64_t>(widest, sl.cols);
    h->item_cap = (std::max<int64_t>(ycols, MAX_T_SLOTS) + 7) / 8 * 8;
    h->pp.tcols_cap = std::max<int64_t>(widest, std::min<int64_t>(op.m, MAX_TCOLS));
    // Y: one t value per column; T: both sources of a merged term's slice
    h->src_cap = std::max<int64_t>(std::max<int64_t>(h->item_cap, yvec), 2 * h->pp.tcols_cap);
    h->pp.item_cap = h->item_cap;
  } else {
    // a dense Y task stages one source vector per kernel term: the most terms
    // any program's task carries (the plan's term structure does not depend
    // on the stage size)
    PlanParams probe;
    probe.half_elems = (int64_t)1 << 30;
    probe.dense_rows_per_task = 1;
    int64_t terms = 1;
    for (const Program& pg : {build_apply_A(op, probe), build_apply_M(op, 2, probe),
                              build_gs_sweep(op, probe)})
      for (const DevTask& t : pg.tasks) terms = std::max<int64_t>(terms, t.nterm);
    h->src_cap = 2 * terms * op.m;  // both sources of every term
    h->item_cap = 0;
  }
  h->blob_cap = (blob_bytes_max(h->item_cap, h->run_cap, h->srun_cap) + 127) / 128 * 128;
  h->slot_bytes =
      h->blob_cap +
      (h->src_cap + EXEC_EPI * EXEC_EPI_SRC + EXEC_TERMS + EXEC_EYES) * (int64_t)sizeof(double2) +
      EXEC_SRCS * (int64_t)sizeof(void*);
  h->slot_bytes = (h->slot_bytes + 127) / 128 * 128;
  // + the consumers' partials (the slot count is settled below)
  size_t fixed = (size_t)EXEC_TSLOTS * h->slot_bytes + EXEC_PART * sizeof(double2);
  // B200 figures for a host-only handle; the device's own otherwise
  int smem_sm = 233472, smem_blk = 232448, reserved = 1024, nsm = 148;
  cudaFuncAttributes fa{};
  fa.sharedSizeBytes = 512;
  if (!host_only) {
    CK(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device));
    CK(cudaDeviceGetAttribute(&smem_blk, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    CK(cudaFuncGetAttributes(&fa, pt_exec_kernel));
    cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, device);
  }
  const int target = 512 / EXEC_CONSUMERS;  // CTAs of EXEC_THREADS per SM
  // ring: 3 stages (PT_STAGES overrides, 2..8; fewer if a stage would not
  // hold `need`).  Items address a stage with 16-bit offsets.
  int max_stages = 3;
  if (const char* e = std::getenv("PT_STAGES"))
    max_stages = std::max(2, std::min(EXEC_MAX_STAGES, std::atoi(e)));
  int64_t half = 0;
  int ctas_sm = 1, stages = 2;
  // Task slots: as many as leave the ring stages room for a full task piece
  // (DENSE_RT_MAX dense kernel rows, or 2048 PLR elements); fewer slots
  // otherwise (big dense slots: c2 at three slots would stage one kernel row
  // per piece).  PT_SLOTS overrides.
  const int64_t want = op.fmt == PT_KERNEL_DENSE ? DENSE_RT_MAX * op.m : std::max<int64_t>(need, 2048);
  int min_slots = 2, max_slots = EXEC_TSLOTS;
  if (const char* e = std::getenv("PT_SLOTS"))
    min_slots = max_slots = std::max(1, std::min(EXEC_TSLOTS, std::atoi(e)));
  for (int ns = max_slots; ns >= min_slots; --ns) {
    h->n_slots = ns;
    fixed = (size_t)ns * h->slot_bytes + EXEC_PART * sizeof(double2);
    half = 0;
    for (int c = target; c >= 1 && half < need; --c) {
      ctas_sm = c;
      const int64_t per_cta =
          std::min<int64_t>(smem_sm / c - reserved - (int64_t)fa.sharedSizeBytes - 128, smem_blk);
      for (stages = max_stages; stages >= 2; --stages) {
        const int64_t hb = (per_cta - (int64_t)fixed) / stages;
        half = hb > 0 ? std::min<int64_t>(65528, (hb / (int64_t)sizeof(double2)) / 8 * 8) : 0;
        if (half >= need) break;
      }
    }
    if (half >= want) break;
  }
  if (half < need) return fail(PT_EINVAL, "block size too large for the executor's shared memory");
  h->pp.half_elems = half;
  h->n_stages = stages;
  h->smem = (size_t)stages * half * sizeof(double2) + fixed;
  if (host_only) {
    h->grid = nsm * ctas_sm;
  } else {
    // the attribute is per function, shared by every handle: it only grows,
    // so a handle with a smaller budget never caps a larger one's launches
    static std::atomic<int> attr_max{0};
    int cur = attr_max.load();
    while ((int)h->smem > cur && !attr_max.compare_exchange_weak(cur, (int)h->smem)) {
    }
    CK(cudaFuncSetAttribute(pt_exec_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                            (int)cudaSharedmemCarveoutMaxShared));
    CK(cudaFuncSetAttribute(pt_exec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            std::max(cur, (int)h->smem)));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pt_exec_kernel, EXEC_THREADS, h->smem));
    if (occ < 1) return fail(PT_EINVAL, "executor kernel does not fit on an SM");
    h->grid = nsm * occ;
  }
  // the queue-order simulation models two tasks in flight per CTA (measured
  // best with three task slots: c3 GMRES 19.5 ms vs 20.4 ms at one or 21.2 at three)
  h->pp.ctas = h->grid * 2;
  // (a PLR operator's Y_DENSE tasks carry no kernel term: identity/rhs rows)
  h->pp.dense_rows_per_task =
      op.fmt == PT_KERNEL_PLR
          ? DENSE_RT_MAX
          : (int)std::max<int64_t>(1, std::min<int64_t>(DENSE_RT_MAX, half / std::max<int64_t>(op.m, 1)));
  h->pp.plr_rows_per_task = PLR_TILE;
  h->pp.plr_slots_per_task = MAX_T_SLOTS;
  if (op.fmt == PT_KERNEL_DENSE) h->pp.item_cap = 0;
  h->pp.t_pieces = want_t_pieces;
  // a ring stage of a Y task may hold two terms' columns (PT_PIECE_PAIRS=0: one term per piece)
  h->pp.piece_pairs = true;
  if (const char* e = std::getenv("PT_PIECE_PAIRS")) h->pp.piece_pairs = std::atoi(e) != 0;
  if (const char* e = std::getenv("PT_DENSE_ROWS"))
    h->pp.dense_rows_per_task = std::max(1, std::min(DENSE_RT_MAX, std::atoi(e)));
  if (const char* e = std::getenv("PT_T_SLOTS")) h->pp.plr_slots_per_task = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("PT_T_PIECES")) h->pp.t_pieces = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("PT_ROW_CHUNK")) h->pp.row_chunk = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("PT_POLL_NS")) h->poll_ns = std::max(0, std::atoi(e));
  if (const char* e = std::getenv("PT_T_PIECES_CHAIN"))
    h->pp.t_pieces_chain = std::max(1, std::atoi(e));
  {
    // Second pass: the blob area was reserved for the largest task the
    // limits allow (EXEC_PIECES pieces, EXEC_TERMS terms, EXEC_WAITS waits);
    // the operator's programs need far less, and what is saved goes to the
    // ring stages.  The programs are planned again with the larger stage and
    // must still fit (a larger stage packs a few more Vt rows into a T
    // task); otherwise the first-pass geometry stays.
    auto max_blob = [&](int64_t* mx) {
      *mx = 0;
      for (const Program& pg : {build_apply_A(op, h->pp), build_apply_M(op, 2, h->pp), build_gs_sweep(op, h->pp)}) {
        if (!pg.overflow.empty()) return false;
        std::vector<int4> blob;
        std::vector<int64_t> off;
        int64_t m1 = 0;
        build_blobs(pg, blob, off, &m1);
        *mx = std::max(*mx, m1);
      }
      return true;
    };
    int64_t mx = 0;
    if (max_blob(&mx)) {
      const int64_t blob2 = (mx + 512 + 127) / 128 * 128;
      if (blob2 < h->blob_cap) {
        const pt_handle::ExecGeom first = h->geom();
        const int64_t slot2 = h->slot_bytes - (h->blob_cap - blob2);
        const int64_t fixed2 = (int64_t)h->n_slots * slot2 + EXEC_PART * (int64_t)sizeof(double2);
        const int64_t half2 = std::min<int64_t>(
            65528, ((int64_t)h->smem - fixed2) / h->n_stages / (int64_t)sizeof(double2) / 8 * 8);
        if (half2 > h->pp.half_elems) {
          h->blob_cap = blob2;
          h->slot_bytes = slot2;
          h->pp.half_elems = half2;
          if (op.fmt == PT_KERNEL_DENSE && !std::getenv("PT_DENSE_ROWS"))
            h->pp.dense_rows_per_task = (int)std::max<int64_t>(
                1, std::min<int64_t>(DENSE_RT_MAX, half2 / std::max<int64_t>(op.m, 1)));
          int64_t mx2 = 0;
          if (!max_blob(&mx2) || mx2 > blob2) h->set_geom(first);
        }
      }
    }
  }
  if (std::getenv("PT_VERBOSE"))
    std::fprintf(stderr, "executor geometry: smem %zu B, %d slots x %lld B (blob %lld, vec %lld), %d stages x %lld B, block terms %d\n",
                 h->smem, h->n_slots, (long long)h->slot_bytes, (long long)h->blob_cap,
                 (long long)h->src_cap * 16, h->n_stages, (long long)h->pp.half_elems * 16,
                 h->pp.max_block_terms);
  return 0;
}

int pt_create(const pt_layout* layout, const pt_entry* entries, int64_t n_entries,
              const int64_t* perm, const double* dense, const pt_leaf* leaves, int64_t n_leaves,
              const double* factors, int64_t n_factor_complex, int device, pt_handle** out) {
  if (!layout || !out || (n_entries > 0 && !entries) || !perm)
    return fail(PT_EINVAL, "null argument to pt_create");
  *out = nullptr;
  const bool host_only = device == PT_DEVICE_HOST;
  if (!host_only) {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(PT_EINVAL, "no such CUDA device");
  }
  std::unique_ptr<DeviceGuard> guard(host_only ? nullptr : new DeviceGuard(device));
  std::unique_ptr<pt_handle> h(new pt_handle());
  h->device = device;
  h->host_only = host_only;
  if (const char* e = std::getenv("PT_DENSE_LEAVES")) h->dense_leaves = std::atoi(e) != 0;
  Operator& op = h->op;
  op.m = layout->m;
  op.nb = layout->n_block_rows;
  op.fmt = layout->kernel_format;
  op.nk = layout->n_kernels;
  if (op.fmt != PT_KERNEL_DENSE && op.fmt != PT_KERNEL_PLR)
    return fail(PT_EINVAL, "unknown kernel format");
  if (op.nk < 0) return fail(PT_EINVAL, "negative kernel count");
  if (op.m > (int64_t)1 << 20) return fail(PT_EINVAL, "block size too large");
  op.perm.assign(perm, perm + std::max<int64_t>(layout->n_block_rows, 0));
  for (int64_t i = 0; i < n_entries; ++i) {
    const pt_entry& e = entries[i];
    op.entries.push_back(HostEntry{e.row, e.col, e.kernel, e.scale_re, e.scale_im, e.eye_re, e.eye_im});
  }
  std::string err;
  if (!validate_operator(op, err)) return fail(PT_EINVAL, err);
  h->sweep_err = sweep_diagonal_error(op);
  int rc;
  h->api_fmt = op.fmt;
  if (op.fmt == PT_KERNEL_DENSE) {
    op.kernel_bytes.assign(op.nk, 16 * op.m * op.m);
    if (op.nk > 0 && !host_only) {
      if (!dense) return fail(PT_EINVAL, "dense kernel array missing");
      const size_t bytes = (size_t)op.nk * op.m * op.m * sizeof(double2);
      CK(cudaMalloc(&h->dense, bytes));
      h->dense_elems = (int64_t)op.nk * op.m * op.m;
      CK(cudaMemcpy(h->dense, dense, bytes, cudaMemcpyHostToDevice));
    }
    // the single-source executor streams dense kernels tile-major, as the
    // dense leaves of a PLR kernel (PT_DENSE_TILES=0: row-major Y_DENSE tasks)
    bool tiles = true;
    if (const char* e = std::getenv("PT_DENSE_TILES")) tiles = std::atoi(e) != 0;
    if (tiles) {
      if ((rc = build_dense_tiles(h.get(), dense))) return rc;
      op.fmt = PT_KERNEL_PLR;
    }
  } else {
    if (n_leaves > 0 && (!leaves || !factors)) return fail(PT_EINVAL, "PLR tables missing");
    if ((rc = build_plr_tables(h.get(), leaves, n_leaves, factors, n_factor_complex))) return rc;
  }
  if (const char* e = std::getenv("PT_BLOCK_TERMS")) h->pp.max_block_terms = std::max(0, std::atoi(e));
  if ((rc = size_executor(h.get(), host_only, device, 4))) return rc;
  if (h->api_fmt == PT_KERNEL_PLR && !std::getenv("PT_BLOCK_TERMS") && !std::getenv("PT_T_PIECES")) {
    // the fused iteration's geometry: block rows as two-term partial sums, T
    // tasks of two ring pieces (see fused_params)
    const pt_handle::ExecGeom base = h->geom();
    h->pp.max_block_terms = 2;
    h->run_cap = h->srun_cap = 0;
    if ((rc = size_executor(h.get(), host_only, device, 2))) return rc;  // (T pieces 1 / 3 measured: 17.75 / 17.05 ms)
    h->fused = h->geom();
    h->has_fused = true;
    h->set_geom(base);
  }
  if (!host_only) CK(cudaMalloc(&h->tmp, std::max<int64_t>(h->N(), 1) * sizeof(double2)));
  if (!host_only && pt_checked_build()) {  // the executor's failure record (mapped host memory)
    CK(cudaHostAlloc(&h->chk_host, 4 * sizeof(long long), cudaHostAllocMapped));
    std::memset(h->chk_host, 0, 4 * sizeof(long long));
    CK(cudaHostGetDevicePointer(&h->chk_dev, h->chk_host, 0));
  }
  *out = h.release();
  return 0;
}

int pt_destroy(pt_handle* h) {
  if (!h) return 0;
  if (h->host_only) {
    delete h;
    return 0;
  }
  DeviceGuard guard(h->device);
  cudaDeviceSynchronize();
  delete h;
  return 0;
}

int pt_apply_A(pt_handle* h, const double* x, double* y, pt_stream stream) {
  if (h && h->host_only) return fail(PT_EINVAL, "plan-only handle (PT_DEVICE_HOST)");
  if (!h || !x || !y) return fail(PT_EINVAL, "null argument");
  DeviceGuard guard(h->device);
  DevProgram* p;
  int rc = get_program(h, "A", 0, &p);
  if (rc) return rc;
  if ((rc = run_program(h, p, (const double2*)x, (double2*)y, nullptr, (cudaStream_t)stream)))
    return rc;
  CK(cudaGetLastError());
  return 0;
}

int pt_apply_M(pt_handle* h, const double* r, double* z, int32_t n_it, pt_stream stream) {
  if (h && h->host_only) return fail(PT_EINVAL, "plan-only handle (PT_DEVICE_HOST)");
  if (!h || !r || !z) return fail(PT_EINVAL, "null argument");
  if (n_it < 1) return fail(PT_EINVAL, "n_it must be at least 1");
  if (!h->sweep_err.empty()) return fail(PT_EINVAL, h->sweep_err);
  DeviceGuard guard(h->device);
  DevProgram* p;
  int rc = get_program(h, "M", n_it, &p);
  if (rc) return rc;
  if ((rc = run_program(h, p, (const double2*)r, (double2*)z, nullptr, (cudaStream_t)stream)))
    return rc;
  CK(cudaGetLastError());
  return 0;
}

int pt_apply_AM(pt_handle* h, const double* x, double* w, int32_t n_it, pt_stream stream) {
  if (h && h->host_only) return fail(PT_EINVAL, "plan-only handle (PT_DEVICE_HOST)");
  if (!h || !x || !w) return fail(PT_EINVAL, "null argument");
  if (n_it < 1) return fail(PT_EINVAL, "n_it must be at least 1");
  if (!h->sweep_err.empty()) return fail(PT_EINVAL, h->sweep_err);
  DeviceGuard guard(h->device);
  DevProgram* p;
  int rc = get_program(h, "AM", n_it, &p);
  if (rc) return rc;
  if ((rc = run_program(h, p, (const double2*)x, (double2*)w, nullptr, (cudaStream_t)stream)))
    return rc;
  CK(cudaGetLastError());
  return 0;
}

int pt_gs_sweep(pt_handle* h, const double* rhs, const double* u_in, double* u_out,
                pt_stream stream) {
  if (h && h->host_only) return fail(PT_EINVAL, "plan-only handle (PT_DEVICE_HOST)");
  if (!h || !rhs || !u_in || !u_out) return fail(PT_EINVAL, "null argument");
  if (!h->sweep_err.empty()) return fail(PT_EINVAL, h->sweep_err);
  DeviceGuard guard(h->device);
  DevProgram* p;
  int rc = get_program(h, "S", 0, &p);
  if (rc) return rc;
  if ((rc = run_program(h, p, (const double2*)rhs, (double2*)u_out, (const double2*)u_in,
                        (cudaStream_t)stream)))
    return rc;
  CK(cudaGetLastError());
  return 0;
}

}  // extern "C"

namespace {

// Build the whole online solve as one CUDA graph:
//   M b -> V0, beta | WHILE(cond) { A->M iteration program on V_j,
//   CGS2 + Givens (sets cond) } | y, x = V y, A x, true residual, D2H status.
// The host synchronises once per solve.
int build_solve_graph(pt_handle* h, int n_it, int max_iter, double tol,
                      pt_handle::SolveGraph* out) {
  DevProgram *pM, *pAM, *pA;
  int rc;
  if ((rc = get_program(h, "M", n_it, &pM))) return rc;
  if ((rc = get_program(h, "AM", n_it, &pAM))) return rc;
  if ((rc = get_program(h, "A", 0, &pA))) return rc;
  pt_gmres_ws* w = h->gws.get();
  GmresDev& d = w->d;
  cudaStream_t cs = h->cap_stream;
  cudaGraph_t g = nullptr, tmp = nullptr;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle cond;
  CK(cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault));
  // kernel launches counted per part; a capture launches nothing, the
  // graph's executions are counted when it runs (gmres_graph)
  const int64_t c0 = g_launches.load();
  // prologue
  CK(cudaStreamBeginCaptureToGraph(cs, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  rc = run_program(h, pM, h->gb, d.V, nullptr, cs);
  if (!rc) gm_begin(d, cond, cs);
  cudaStreamCaptureStatus cst;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  cudaError_t ce = cudaStreamGetCaptureInfo(cs, &cst, nullptr, nullptr, &deps, &ndeps);
  std::vector<cudaGraphNode_t> tail(deps, deps + ndeps);
  CK(cudaStreamEndCapture(cs, &tmp));
  if (rc) return rc;
  CK(ce);
  // loop
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = cond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t loop;
  CK(cudaGraphAddNode(&loop, g, tail.data(), tail.size(), &cp));
  const int64_t c1n = g_launches.load();
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal));
  IterMode im;
  im.iter = &d.st->iterations;
  im.vbase = d.V;
  im.vstride = d.n;
  rc = run_program(h, pAM, nullptr, nullptr, nullptr, cs, &d.st->stop, im);
  cudaError_t ae = rc ? cudaSuccess : gm_arnoldi_step(d, tol, max_iter, cond, cs);
  CK(cudaStreamEndCapture(cs, &tmp));
  if (rc) return rc;
  CK(ae);
  const int64_t c2n = g_launches.load();
  // epilogue
  CK(cudaStreamBeginCaptureToGraph(cs, g, &loop, nullptr, 1, cudaStreamCaptureModeThreadLocal));
  gm_finish(d, h->gx, cs);
  rc = run_program(h, pA, h->gx, h->tmp, nullptr, cs);
  if (!rc) gm_resid(d, h->gb, h->tmp, cs);
  cudaError_t c1 = cudaMemcpyAsync(w->st_host, d.st, sizeof(DevStatus), cudaMemcpyDeviceToHost, cs);
  cudaError_t c2 = cudaMemcpyAsync(h->hist_host, d.hist, (size_t)max_iter * sizeof(double),
                                   cudaMemcpyDeviceToHost, cs);
  CK(cudaStreamEndCapture(cs, &tmp));
  if (rc) return rc;
  CK(c1);
  CK(c2);
  CK(cudaGraphInstantiate(&out->exec, g, 0));
  CK(cudaGraphDestroy(g));
  const int64_t c3n = g_launches.load();
  out->k_pro = c1n - c0;
  out->k_body = c2n - c1n;
  out->k_epi = c3n - c2n;
  g_launches.fetch_sub(c3n - c0);
  out->n_it = n_it;
  out->max_iter = max_iter;
  out->tol = tol;
  return 0;
}

int finish_report(pt_handle* h, const DevStatus& st, int max_iter, pt_report* rep) {
  fill_report(st, rep);
  if (st.nonfinite) {
    rep->nonfinite = 1;
    return fail(PT_ENONFINITE, "non-finite values in preconditioned matvec at iteration " +
                                   std::to_string(st.iterations + 1));
  }
  if (st.beta == 0.0) {  // solver.py:239-242
    rep->converged = 1;
    rep->flag = PT_FLAG_CONVERGED;
    rep->true_residual = 0.0;
    return 0;
  }
  const double tr = std::sqrt(st.true_num2), sc = std::sqrt(st.b_norm2);
  rep->true_residual = sc > 0.0 ? tr / sc : tr;
  (void)h;
  (void)max_iter;
  return 0;
}

// Graph path: b/x may be the graph's own buffers (then no copies).
int gmres_graph(pt_handle* h, const double2* b, double2* x, bool b_host, bool x_host,
                const pt_gmres_config* cfg, pt_report* rep, cudaStream_t s) {
  int rc;
  if ((rc = ensure_gws(h, cfg->max_iter))) return rc;
  const int64_t N = h->N();
  const size_t bytes = (size_t)N * sizeof(double2);
  if (!h->cap_stream) CK(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
  if (!h->gb) CK(cudaMalloc(&h->gb, bytes));
  if (!h->gx) CK(cudaMalloc(&h->gx, bytes));
  // programs first: building them may reallocate buffers (and drop graphs)
  DevProgram* p;
  if ((rc = get_program(h, "M", cfg->n_it, &p))) return rc;
  if ((rc = get_program(h, "AM", cfg->n_it, &p))) return rc;
  if ((rc = get_program(h, "A", 0, &p))) return rc;
  pt_handle::SolveGraph* sg = nullptr;
  for (auto& g : h->graphs)
    if (g.n_it == cfg->n_it && g.max_iter == cfg->max_iter && g.tol == cfg->rel_tol) sg = &g;
  if (!sg) {
    pt_handle::SolveGraph ng;
    if ((rc = build_solve_graph(h, cfg->n_it, cfg->max_iter, cfg->rel_tol, &ng))) return rc;
    h->graphs.push_back(ng);
    sg = &h->graphs.back();
  }
  if (b != h->gb)
    CK(cudaMemcpyAsync(h->gb, b, bytes, b_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                       s));
  CK(cudaGraphLaunch(sg->exec, s));
  if (x != h->gx)
    CK(cudaMemcpyAsync(x, h->gx, bytes, x_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                       s));
  CK(cudaStreamSynchronize(s));
  const DevStatus st = h->gws->st_host[0];
  // kernels the graph ran: prologue, one body per iteration, epilogue
  g_launches.fetch_add(sg->k_pro + (int64_t)st.iterations * sg->k_body + sg->k_epi);
  if (rep->residual_history && st.iterations > 0)
    std::memcpy(rep->residual_history, h->hist_host, (size_t)st.iterations * sizeof(double));
  return finish_report(h, st, cfg->max_iter, rep);
}

// Host-driven path (PT_GRAPH=0, and whenever per-launch timing is on):
// iterations are enqueued speculatively one batch ahead of the host's
// convergence check; kernels after the stop return immediately.
int gmres_stream(pt_handle* h, const double2* b, double2* x, const pt_gmres_config* cfg,
                 pt_report* rep, cudaStream_t s) {
  int rc;
  if ((rc = ensure_gws(h, cfg->max_iter))) return rc;
  pt_gmres_ws* w = h->gws.get();
  GmresDev& d = w->d;
  DevProgram *pM, *pAM, *pA;
  if ((rc = get_program(h, "M", cfg->n_it, &pM))) return rc;
  if ((rc = get_program(h, "AM", cfg->n_it, &pAM))) return rc;
  if ((rc = get_program(h, "A", 0, &pA))) return rc;
  const int64_t N = h->N();
  if ((rc = run_program(h, pM, b, d.V, nullptr, s))) return rc;
  gm_begin(d, 0, s);
  // per-launch timing: one iteration per batch and no speculative launches
  // (a launch after the stop returns at once but would still be counted with
  // its program's bytes)
  const bool ahead = !h->timing;
  const int B = ahead ? 2 : 1;
  int enq = 0, nb = 0, waited = 0;
  DevStatus last{};
  IterMode im;
  im.iter = &d.st->iterations;
  im.vbase = d.V;
  im.vstride = N;
  auto enqueue_batch = [&]() -> int {
    for (int i = 0; i < B && enq < cfg->max_iter; ++i, ++enq) {
      int r = run_program(h, pAM, nullptr, nullptr, nullptr, s, &d.st->stop, im);
      if (r) return r;
      CK(gm_arnoldi_step(d, cfg->rel_tol, cfg->max_iter, 0, s));
    }
    CK(cudaMemcpyAsync(w->st_host + (nb % 2), d.st, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(w->ev[nb % 2], s));
    ++nb;
    return 0;
  };
  if ((rc = enqueue_batch())) return rc;
  for (;;) {
    if (ahead && enq < cfg->max_iter && (rc = enqueue_batch())) return rc;
    CK(cudaEventSynchronize(w->ev[waited % 2]));
    last = w->st_host[waited % 2];
    ++waited;
    if (last.stop) break;
    if (!ahead && enq < cfg->max_iter) {
      if ((rc = enqueue_batch())) return rc;
      continue;
    }
    if (waited == nb && enq >= cfg->max_iter) break;
  }
  gm_finish(d, x, s);
  if ((rc = run_program(h, pA, x, h->tmp, nullptr, s))) return rc;
  gm_resid(d, b, h->tmp, s);
  CK(cudaGetLastError());
  if ((rc = fetch_status(w, s))) return rc;
  const DevStatus st = *w->st_host;
  if (rep->residual_history && st.iterations > 0)
    CK(cudaMemcpy(rep->residual_history, d.hist, (size_t)st.iterations * sizeof(double),
                  cudaMemcpyDeviceToHost));
  return finish_report(h, st, cfg->max_iter, rep);
}

bool use_graph(const pt_handle* h) {
  const char* e = std::getenv("PT_GRAPH");
  return !h->timing && !(e && e[0] == '0');
}

// ---- multi-RHS (batched) path ------------------------------------------------
// Dense operators only: the batched executor streams dense kernel rows (a
// PLR operator keeps the per-source solves, see pt_gmres_batch).

int batch_init(pt_handle* h) {
  auto& B = h->batch;
  if (B.grid > 0) return 0;
  CK(bexec_setup());
  CK(bg_setup(1));
  if (const char* e = std::getenv("PT_BATCH_ROWS")) B.rows = std::atoi(e) == 16 ? 16 : 8;
  if (const char* e = std::getenv("PT_BATCH_COLS")) B.tcols = std::atoi(e) == 64 ? BW : 32;
  if (std::getenv("PT_BATCH_ROWS") && !std::getenv("PT_BATCH_COLS")) B.tcols = BW;
  if (B.tcols == 32) B.rows = 16;  // the 16 x 32 tile
  B.grid = bexec_grid(h->device, B.rows, B.tcols);
  if (B.grid <= 0) return fail(PT_ECUDA, "batched executor does not fit on an SM");
  B.pp = h->pp;
  B.pp.force_dense = true;  // Y_DENSE tasks over the row-major dense pool
  B.pp.max_block_terms = 0;
  B.pp.ctas = B.grid;
  B.pp.dense_rows_per_task = B.rows;
  B.pp.row_chunk = B.rows;  // every task its own producer group: finest dependencies
  B.pp.half_elems = (int64_t)B.rows * h->op.m;
  // list-scheduling model: a task's cost is its kernel bytes at the
  // FP64-bound rate of one CTA (BW/2 flop per kernel byte)
  B.pp.task_us = 1.0;
  B.pp.cta_gbs = 2.5;
  const size_t bytes = (size_t)h->N() * BW * sizeof(double2);
  CK(cudaMalloc(&B.b, bytes));
  CK(cudaMalloc(&B.x, bytes));
  CK(cudaMalloc(&B.tmp, bytes));
  CK(cudaMalloc(&B.cols, bytes));
  CK(cudaMemset(B.b, 0, bytes));
  CK(cudaMemset(B.x, 0, bytes));
  for (auto& e : B.ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return 0;
}

int ensure_bslot(pt_handle* h, int s, int64_t elems) {
  auto& B = h->batch;
  if (elems <= B.slot_cap[s]) return 0;
  CK(cudaDeviceSynchronize());
  B.drop_graphs();
  cudaFree(B.slot[s]);
  CK(cudaMalloc(&B.slot[s], (size_t)elems * BW * sizeof(double2)));
  CK(cudaMemset(B.slot[s], 0, (size_t)elems * BW * sizeof(double2)));
  B.slot_cap[s] = elems;
  return 0;
}

int get_bprogram(pt_handle* h, const std::string& kind, int n_it, DevProgram** out) {
  auto& B = h->batch;
  int rc;
  if ((rc = batch_init(h))) return rc;
  const std::string key = kind + std::to_string(n_it);
  auto it = B.progs.find(key);
  if (it != B.progs.end()) {
    *out = it->second.get();
    return 0;
  }
  std::unique_ptr<DevProgram> p(new DevProgram());
  p->fused = kind == "AM" && h->has_fused;
  FusedGeom scope(h, p->fused);
  if (kind == "A")
    p->host = build_apply_A(h->op, B.pp);
  else if (kind == "M")
    p->host = build_apply_M(h->op, n_it, B.pp);
  else
    p->host = build_A_then_M(h->op, n_it, B.pp);
  if (!p->host.overflow.empty()) return fail(PT_EINVAL, p->host.overflow);
  for (const DevTask& t : p->host.tasks)
    if (t.type != TASK_Y_DENSE || t.nterm > BT_TERMS || t.neye > BT_EYES || t.r1 - t.r0 > B.rows)
      return fail(PT_EINVAL, "a task exceeds what the batched executor stages");
  if (B.tcols < BW) {
    // every task becomes BW / tcols tasks over disjoint source columns (same
    // waits; each producer group counts all of them)
    const int split = BW / B.tcols;
    std::vector<DevTask> tasks;
    for (const DevTask& t : p->host.tasks)
      for (int c = 0; c < split; ++c) {
        DevTask u = t;
        u.c0 = c * B.tcols;
        u.c1 = u.c0 + B.tcols;
        tasks.push_back(u);
      }
    p->host.tasks.swap(tasks);
    for (DevWait& w : p->host.waits) w.val *= split;
  }
  if ((rc = upload(&p->tasks, p->host.tasks))) return rc;
  if ((rc = upload(&p->terms, p->host.terms))) return rc;
  if ((rc = upload(&p->eyes, p->host.eyes))) return rc;
  if ((rc = upload(&p->waits, p->host.waits))) return rc;
  for (int s : {SLOT_Y, SLOT_U1, SLOT_U2, SLOT_PRE})
    if ((rc = ensure_bslot(h, s, p->host.slot_elems[s]))) return rc;
  if (p->host.n_counters + 1 > B.ctr_cap) {
    CK(cudaDeviceSynchronize());
    B.drop_graphs();
    cudaFree(B.ctr);
    B.ctr_cap = p->host.n_counters + 1;
    CK(cudaMalloc(&B.ctr, B.ctr_cap * sizeof(int)));
  }
  *out = p.get();
  B.progs[key] = std::move(p);
  return 0;
}

int run_bprogram(pt_handle* h, DevProgram* p, const double2* in, double2* out, cudaStream_t s,
                 const int* stop = nullptr, const int* iter = nullptr, double2* vbase = nullptr,
                 int64_t vstride = 0) {
  auto& B = h->batch;
  if (p->host.tasks.empty()) return 0;
  BExecArgs a{};
  a.tasks = p->tasks;
  a.terms = p->terms;
  a.eyes = p->eyes;
  a.waits = p->waits;
  a.ctr = B.ctr;
  a.head = B.ctr + p->host.n_counters;
  for (int i = 0; i < N_SLOTS; ++i) a.slot[i] = B.slot[i];
  a.slot[SLOT_IN] = const_cast<double2*>(in);
  a.slot[SLOT_OUT] = out;
  a.dense = h->dense;
  a.n_tasks = (int)p->host.tasks.size();
  a.m = (int)h->op.m;
  a.stop = stop;
  a.iter = iter;
  a.vbase = vbase;
  a.vstride = vstride;
  if (int orc = order_before(h, s)) return orc;
  CK(cudaMemsetAsync(B.ctr, 0, (p->host.n_counters + 1) * sizeof(int), s));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (h->timing) {
    for (cudaEvent_t* e : {&e0, &e1}) {
      if (h->ev_free.empty()) {
        CK(cudaEventCreate(e));
      } else {
        *e = h->ev_free.back();
        h->ev_free.pop_back();
      }
    }
    CK(cudaEventRecord(e0, s));
  }
  CK(bexec_launch(a, B.grid, B.rows, B.tcols, s));
  if (int orc = order_after(h, s)) return orc;
  if (h->timing) {
    CK(cudaEventRecord(e1, s));
    h->ev_used.emplace_back(e0, e1);
    h->timed_launches += 1;
    h->timed_bytes += p->host.algo_bytes;
  }
  return 0;
}

int ensure_bgws(pt_handle* h, int max_iter) {
  auto& B = h->batch;
  if (B.g_iter >= max_iter) return 0;
  CK(cudaDeviceSynchronize());
  B.drop_graphs();
  B.free_gmres();
  BGmresDev& g = B.g;
  const int64_t N = h->N();
  const size_t ldr = (size_t)max_iter + 1;
  g.n = N;
  g.max_iter = max_iter;
  CK(cudaMalloc(&g.V, ldr * N * BW * sizeof(double2)));
  CK(cudaMalloc(&g.P, (size_t)BRED_BLOCKS * ldr * BW * sizeof(double2)));
  CK(cudaMalloc(&g.h1, ldr * BW * sizeof(double2)));
  CK(cudaMalloc(&g.h2, ldr * BW * sizeof(double2)));
  CK(cudaMalloc(&g.R, (size_t)BW * ldr * max_iter * sizeof(double2)));
  CK(cudaMalloc(&g.g, (size_t)BW * ldr * sizeof(double2)));
  CK(cudaMalloc(&g.cs, (size_t)BW * max_iter * sizeof(double)));
  CK(cudaMalloc(&g.sn, (size_t)BW * max_iter * sizeof(double2)));
  CK(cudaMalloc(&g.hist, (size_t)BW * max_iter * sizeof(double)));
  CK(cudaMalloc(&g.y, (size_t)BW * max_iter * sizeof(double2)));
  CK(cudaMalloc(&g.inv, BW * sizeof(double)));
  CK(cudaMalloc(&g.st, BW * sizeof(DevStatus)));
  CK(cudaMalloc(&g.ctl, 4 * sizeof(int)));
  CK(cudaMemset(g.V, 0, ldr * N * BW * sizeof(double2)));
  CK(cudaMemset(g.st, 0, BW * sizeof(DevStatus)));
  CK(cudaMemset(g.ctl, 0, 4 * sizeof(int)));
  CK(cudaMallocHost(&B.st_host, BW * sizeof(DevStatus)));
  CK(cudaMallocHost(&B.hist_host, (size_t)BW * max_iter * sizeof(double)));
  CK(cudaMallocHost(&B.ctl_host, 2 * 4 * sizeof(int)));
  CK(bg_setup(max_iter));
  B.g_iter = max_iter;
  return 0;
}

// One batch of up to BW sources, already packed into B.b; solution in B.x,
// statuses and histories in the pinned host arrays.  Whole solve as one CUDA
// graph (conditional WHILE over the lockstep iterations) unless per-launch
// timing is on; then a host loop one step ahead of its stop check.
int bgmres_run(pt_handle* h, const pt_gmres_config* cfg, int nrhs, cudaStream_t s) {
  auto& B = h->batch;
  int rc;
  DevProgram *pM, *pAM, *pA;
  if ((rc = get_bprogram(h, "M", cfg->n_it, &pM))) return rc;
  if ((rc = get_bprogram(h, "AM", cfg->n_it, &pAM))) return rc;
  if ((rc = get_bprogram(h, "A", 0, &pA))) return rc;
  if ((rc = ensure_bgws(h, cfg->max_iter))) return rc;
  BGmresDev g = B.g;
  g.max_iter = B.g_iter;
  g.nrhs = nrhs;
  const int64_t N = h->N();
  const int64_t vstride = N * BW;
  auto epilogue = [&](cudaStream_t cs) -> int {
    bg_finish(g, B.x, cs);
    int r = run_bprogram(h, pA, B.x, B.tmp, cs);
    if (r) return r;
    bg_resid(g, B.b, B.tmp, cs);
    CK(cudaMemcpyAsync(B.st_host, g.st, BW * sizeof(DevStatus), cudaMemcpyDeviceToHost, cs));
    CK(cudaMemcpyAsync(B.hist_host, g.hist, (size_t)BW * g.max_iter * sizeof(double),
                       cudaMemcpyDeviceToHost, cs));
    return 0;
  };
  if (!use_graph(h)) {
    if ((rc = run_bprogram(h, pM, B.b, g.V, s))) return rc;
    bg_begin(g, 0, s);
    int enq = 0, nb = 0, waited = 0;
    // per-launch timing: no speculative launches (see gmres_stream)
    const bool ahead = !h->timing;
    auto enqueue = [&]() -> int {
      for (int i = 0; i < (ahead ? 2 : 1) && enq < cfg->max_iter; ++i, ++enq) {
        int r = run_bprogram(h, pAM, nullptr, nullptr, s, g.ctl + 1, g.ctl, g.V, vstride);
        if (r) return r;
        bg_step(g, cfg->rel_tol, cfg->max_iter, 0, s);
      }
      CK(cudaMemcpyAsync(B.ctl_host + 4 * (nb % 2), g.ctl, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
      CK(cudaEventRecord(B.ev[nb % 2], s));
      ++nb;
      return 0;
    };
    if ((rc = enqueue())) return rc;
    for (;;) {
      if (ahead && enq < cfg->max_iter && (rc = enqueue())) return rc;
      CK(cudaEventSynchronize(B.ev[waited % 2]));
      const int stop = B.ctl_host[4 * (waited % 2) + 1];
      ++waited;
      if (stop) break;
      if (!ahead && enq < cfg->max_iter) {
        if ((rc = enqueue())) return rc;
        continue;
      }
      if (waited == nb && enq >= cfg->max_iter) break;
    }
    if ((rc = epilogue(s))) return rc;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    return 0;
  }
  pt_handle::Batch::Graph* gr = nullptr;
  for (auto& x : B.graphs)
    if (x.n_it == cfg->n_it && x.max_iter == cfg->max_iter && x.tol == cfg->rel_tol && x.nrhs == nrhs)
      gr = &x;
  if (!gr) {
    if (!h->cap_stream) CK(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
    cudaStream_t cs = h->cap_stream;
    cudaGraph_t graph = nullptr, tmp = nullptr;
    CK(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle cond;
    CK(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
    const int64_t c0 = g_launches.load();
    CK(cudaStreamBeginCaptureToGraph(cs, graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    rc = run_bprogram(h, pM, B.b, g.V, cs);
    if (!rc) bg_begin(g, cond, cs);
    cudaStreamCaptureStatus cst;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    cudaError_t ce = cudaStreamGetCaptureInfo(cs, &cst, nullptr, nullptr, &deps, &ndeps);
    std::vector<cudaGraphNode_t> tail(deps, deps + ndeps);
    CK(cudaStreamEndCapture(cs, &tmp));
    if (rc) return rc;
    CK(ce);
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t loop;
    CK(cudaGraphAddNode(&loop, graph, tail.data(), tail.size(), &cp));
    const int64_t c1 = g_launches.load();
    CK(cudaStreamBeginCaptureToGraph(cs, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                     cudaStreamCaptureModeThreadLocal));
    rc = run_bprogram(h, pAM, nullptr, nullptr, cs, g.ctl + 1, g.ctl, g.V, vstride);
    if (!rc) bg_step(g, cfg->rel_tol, cfg->max_iter, cond, cs);
    CK(cudaStreamEndCapture(cs, &tmp));
    if (rc) return rc;
    const int64_t c2 = g_launches.load();
    CK(cudaStreamBeginCaptureToGraph(cs, graph, &loop, nullptr, 1, cudaStreamCaptureModeThreadLocal));
    rc = epilogue(cs);
    CK(cudaStreamEndCapture(cs, &tmp));
    if (rc) return rc;
    pt_handle::Batch::Graph ng;
    CK(cudaGraphInstantiate(&ng.exec, graph, 0));
    CK(cudaGraphDestroy(graph));
    const int64_t c3 = g_launches.load();
    ng.k_pro = c1 - c0;
    ng.k_body = c2 - c1;
    ng.k_epi = c3 - c2;
    g_launches.fetch_sub(c3 - c0);
    ng.n_it = cfg->n_it;
    ng.max_iter = cfg->max_iter;
    ng.tol = cfg->rel_tol;
    ng.nrhs = nrhs;
    B.graphs.push_back(ng);
    gr = &B.graphs.back();
  }
  CK(cudaGraphLaunch(gr->exec, s));
  CK(cudaStreamSynchronize(s));
  int iters = 0;
  for (int k = 0; k < BW; ++k) iters = std::max(iters, B.st_host[k].iterations);
  g_launches.fetch_add(gr->k_pro + (int64_t)iters * gr->k_body + gr->k_epi);
  return 0;
}

// per-source reports of the last batch (sources [0, nrhs)); PT_ENONFINITE if
// any source met non-finite values
int bgmres_reports(pt_handle* h, int nrhs, int max_iter, int first, pt_report* reports) {
  auto& B = h->batch;
  int bad = -1;
  for (int k = 0; k < nrhs; ++k) {
    const DevStatus& st = B.st_host[k];
    if (st.nonfinite && bad < 0) bad = k;
    if (!reports) continue;
    pt_report* rep = reports + first + k;
    double* hist = rep->residual_history;
    *rep = pt_report{};
    rep->residual_history = hist;
    fill_report(st, rep);
    if (hist && st.iterations > 0)
      std::memcpy(hist, B.hist_host + (size_t)k * B.g_iter, (size_t)st.iterations * sizeof(double));
    if (st.beta == 0.0) {
      rep->converged = 1;
      rep->flag = PT_FLAG_CONVERGED;
      rep->true_residual = 0.0;
    } else {
      const double tr = std::sqrt(st.true_num2), sc = std::sqrt(st.b_norm2);
      rep->true_residual = sc > 0.0 ? tr / sc : tr;
    }
  }
  (void)max_iter;
  if (bad >= 0)
    return fail(PT_ENONFINITE, "non-finite values in preconditioned matvec at iteration " +
                                   std::to_string(B.st_host[bad].iterations + 1) + " (source " +
                                   std::to_string(first + bad) + ")");
  return 0;
}

// batched solve of nrhs column-major sources (device or host buffers)
int gmres_batched(pt_handle* h, const double2* b, double2* x, int nrhs, bool host,
                  const pt_gmres_config* cfg, pt_report* reports, cudaStream_t s) {
  int rc;
  if ((rc = batch_init(h))) return rc;
  auto& B = h->batch;
  const int64_t N = h->N();
  int status = 0;
  for (int first = 0; first < nrhs; first += BW) {
    const int nb = std::min(BW, nrhs - first);
    const double2* src = b + (size_t)first * N;
    if (host) {
      CK(cudaMemcpyAsync(B.cols, src, (size_t)nb * N * sizeof(double2), cudaMemcpyHostToDevice, s));
      src = B.cols;
    }
    b_pack(src, N, nb, B.b, s);
    CK(cudaGetLastError());
    if ((rc = bgmres_run(h, cfg, nb, s))) return rc;
    double2* dst = host ? B.cols : x + (size_t)first * N;
    b_unpack(B.x, N, nb, dst, s);
    CK(cudaGetLastError());
    if (host)
      CK(cudaMemcpyAsync(x + (size_t)first * N, B.cols, (size_t)nb * N * sizeof(double2),
                         cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    rc = bgmres_reports(h, nb, cfg->max_iter, first, reports);
    if (rc && !status) status = rc;
  }
  return status;
}

// batched apply of kind "A" or "M" to nrhs column-major device vectors
int apply_batched(pt_handle* h, const std::string& kind, int n_it, const double2* in, double2* out,
                  int nrhs, cudaStream_t s) {
  int rc;
  DevProgram* p;
  if ((rc = get_bprogram(h, kind, n_it, &p))) return rc;
  auto& B = h->batch;
  const int64_t N = h->N();
  for (int first = 0; first < nrhs; first += BW) {
    const int nb = std::min(BW, nrhs - first);
    b_pack(in + (size_t)first * N, N, nb, B.b, s);
    if ((rc = run_bprogram(h, p, B.b, B.tmp, s))) return rc;
    b_unpack(B.tmp, N, nb, out + (size_t)first * N, s);
    CK(cudaGetLastError());
  }
  return 0;
}


}  // namespace

extern "C" {

int pt_gmres(pt_handle* h, const double* b, double* x, const pt_gmres_config* cfg,
             pt_report* report, pt_stream stream) {
  if (h && h->host_only) return fail(PT_EINVAL, "plan-only handle (PT_DEVICE_HOST)");
  if (!h || !b || !x) return fail(PT_EINVAL, "null argument");
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (!h->sweep_err.empty()) return fail(PT_EINVAL, h->sweep_err);
  DeviceGuard guard(h->device);
  pt_report local{};
  pt_report* rep = report ? report : &local;
  double* hist = rep->residual_history;
  *rep = pt_report{};
  rep->residual_history = hist;
  if (use_graph(h))
    return gmres_graph(h, (const double2*)b, (double2*)x, false, false, cfg, rep,
                       (cudaStream_t)stream);
  return gmres_stream(h, (const double2*)b, (double2*)x, cfg, rep, (cudaStream_t)stream);
}

int pt_gmres_host(pt_handle* h, const double* b_host, double* x_host, const pt_gmres_config* cfg,
                  pt_report* report, pt_stream stream) {
  if (h && h->host_only) return fail(PT_EINVAL, "plan-only handle (PT_DEVICE_HOST)");
  if (!h || !b_host || !x_host) return fail(PT_EINVAL, "null argument");
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (!h->sweep_err.empty()) return fail(PT_EINVAL, h->sweep_err);
  DeviceGuard guard(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  pt_report local{};
  pt_report* rep = report ? report : &local;
  double* hist = rep->residual_history;
  *rep = pt_report{};
  rep->residual_history = hist;
  if (use_graph(h))
    return gmres_graph(h, (const double2*)b_host, (double2*)x_host, true, true, cfg, rep, s);
  const size_t bytes = (size_t)h->N() * sizeof(double2);
  if (!h->hb) CK(cudaMalloc(&h->hb, bytes));
  if (!h->hx) CK(cudaMalloc(&h->hx, bytes));
  CK(cudaMemcpyAsync(h->hb, b_host, bytes, cudaMemcpyHostToDevice, s));
  if ((rc = gmres_stream(h, h->hb, h->hx, cfg, rep, s))) return rc;
  CK(cudaMemcpyAsync(x_host, h->hx, bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}

int pt_gmres_batch(pt_handle* h, const double* b, double* x, int32_t nrhs,
                   const pt_gmres_config* cfg, pt_report* reports, pt_stream stream) {
  if (h && h->host_only) return fail(PT_EINVAL, "plan-only handle (PT_DEVICE_HOST)");
  if (!h || !b || !x || nrhs < 0) return fail(PT_EINVAL, "bad argument");
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (!h->sweep_err.empty()) return fail(PT_EINVAL, h->sweep_err);
  const int64_t N = h->N();
  if (h->api_fmt == PT_KERNEL_DENSE && nrhs > 1 && !std::getenv("PT_BATCH_SEQ")) {
    DeviceGuard guard(h->device);
    return gmres_batched(h, (const double2*)b, (double2*)x, nrhs, false, cfg, reports,
                         (cudaStream_t)stream);
  }
  for (int32_t r = 0; r < nrhs; ++r) {
    rc = pt_gmres(h, b + 2 * r * N, x + 2 * r * N, cfg, reports ? reports + r : nullptr, stream);
    if (rc) return rc;
  }
  return 0;
}

int pt_gmres_batch_host(pt_handle* h, const double* b_host, double* x_host, int32_t nrhs,
                        const pt_gmres_config* cfg, pt_report* reports, pt_stream stream) {
  if (h && h->host_only) return fail(PT_EINVAL, "plan-only handle (PT_DEVICE_HOST)");
  if (!h || !b_host || !x_host || nrhs < 0) return fail(PT_EINVAL, "bad argument");
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (!h->sweep_err.empty()) return fail(PT_EINVAL, h->sweep_err);
  const int64_t N = h->N();
  if (h->api_fmt == PT_KERNEL_DENSE && nrhs > 1 && !std::getenv("PT_BATCH_SEQ")) {
    DeviceGuard guard(h->device);
    return gmres_batched(h, (const double2*)b_host, (double2*)x_host, nrhs, true, cfg, reports,
                         (cudaStream_t)stream);
  }
  for (int32_t r = 0; r < nrhs; ++r) {
    rc = pt_gmres_host(h, b_host + 2 * r * N, x_host + 2 * r * N, cfg, reports ? reports + r : nullptr,
                       stream);
    if (rc) return rc;
  }
  return 0;
}

int pt_apply_A_batch(pt_handle* h, const double* x, double* y, int32_t nrhs, pt_stream stream) {
  if (h && h->host_only) return fail(PT_EINVAL, "plan-only handle (PT_DEVICE_HOST)");
  if (!h || !x || !y || nrhs < 0) return fail(PT_EINVAL, "bad argument");
  if (h->api_fmt != PT_KERNEL_DENSE) return fail(PT_EINVAL, "batched applies need a dense operator");
  DeviceGuard guard(h->device);
  return apply_batched(h, "A", 0, (const double2*)x, (double2*)y, nrhs, (cudaStream_t)stream);
}

int pt_apply_M_batch(pt_handle* h, const double* r, double* z, int32_t nrhs, int32_t n_it,
                     pt_stream stream) {
  if (h && h->host_only) return fail(PT_EINVAL, "plan-only handle (PT_DEVICE_HOST)");
  if (!h || !r || !z || nrhs < 0) return fail(PT_EINVAL, "bad argument");
  if (n_it < 1) return fail(PT_EINVAL, "n_it must be at least 1");
  if (!h->sweep_err.empty()) return fail(PT_EINVAL, h->sweep_err);
  if (h->api_fmt != PT_KERNEL_DENSE) return fail(PT_EINVAL, "batched applies need a dense operator");
  DeviceGuard guard(h->device);
  return apply_batched(h, "M", n_it, (const double2*)r, (double2*)z, nrhs, (cudaStream_t)stream);
}

int pt_gmres_ws_create(int64_t n, int32_t max_iter, int device, pt_gmres_ws** out) {
  if (!out || n < 1 || max_iter < 1) return fail(PT_EINVAL, "bad GMRES workspace size");
  DeviceGuard guard(device);
  std::unique_ptr<pt_gmres_ws> w(new pt_gmres_ws());
  w->device = device;
  int rc = ws_alloc(w.get(), n, max_iter);
  if (rc) return rc;
  *out = w.release();
  return 0;
}

int pt_gmres_ws_destroy(pt_gmres_ws* ws) {
  if (!ws) return 0;
  DeviceGuard guard(ws->device);
  cudaDeviceSynchronize();
  delete ws;
  return 0;
}

double* pt_gmres_ws_basis(pt_gmres_ws* ws, int32_t j) {
  if (!ws || j < 0 || j > ws->d.max_iter) return nullptr;
  return (double*)(ws->d.V + (int64_t)j * ws->d.n);
}

int pt_gmres_ws_begin(pt_gmres_ws* ws, const double* mb, double* beta_out, pt_stream stream) {
  if (!ws || !mb) return fail(PT_EINVAL, "null argument");
  DeviceGuard guard(ws->device);
  return ws_begin_impl(ws, mb, beta_out, (cudaStream_t)stream, true);
}

int pt_gmres_ws_step(pt_gmres_ws* ws, int32_t j, double rel_tol, int32_t max_iter,
                     pt_report* report, int32_t* stop_out, pt_stream stream) {
  if (!ws || !stop_out) return fail(PT_EINVAL, "null argument");
  DeviceGuard guard(ws->device);
  int stop = 0;
  int rc = ws_step_impl(ws, j, rel_tol, max_iter, report, &stop, (cudaStream_t)stream);
  *stop_out = stop;
  return rc;
}

int pt_gmres_ws_finish(pt_gmres_ws* ws, int32_t k, double* x, pt_stream stream) {
  if (!ws || !x || k < 0 || k > ws->d.max_iter) return fail(PT_EINVAL, "bad argument");
  DeviceGuard guard(ws->device);
  cudaStream_t s = (cudaStream_t)stream;
  (void)k;  // k is the device's own iteration count (st->iterations)
  gm_finish(ws->d, (double2*)x, s);
  CK(cudaGetLastError());
  return 0;
}

int pt_exec_timing(pt_handle* h, int32_t enable) {
  if (h && h->host_only) return fail(PT_EINVAL, "plan-only handle (PT_DEVICE_HOST)");
  if (!h) return fail(PT_EINVAL, "null handle");
  DeviceGuard guard(h->device);
  double ms;
  int64_t n, b;
  int rc = pt_exec_stats(h, &ms, &n, &b);
  h->timing = enable != 0;
  return rc;
}

int pt_exec_stats(pt_handle* h, double* total_ms, int64_t* launches, int64_t* algo_bytes) {
  if (h && h->host_only) return fail(PT_EINVAL, "plan-only handle (PT_DEVICE_HOST)");
  if (!h) return fail(PT_EINVAL, "null handle");
  DeviceGuard guard(h->device);
  CK(cudaDeviceSynchronize());
  double tot = 0.0;
  for (auto& p : h->ev_used) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, p.first, p.second));
    tot += ms;
    h->ev_free.push_back(p.first);
    h->ev_free.push_back(p.second);
  }
  h->ev_used.clear();
  if (total_ms) *total_ms = tot;
  if (launches) *launches = h->timed_launches;
  if (algo_bytes) *algo_bytes = h->timed_bytes;
  h->timed_launches = 0;
  h->timed_bytes = 0;
  return 0;
}

int pt_trace_program(pt_handle* h, int32_t kind, int32_t n_it, const double* in, double* out,
                     int64_t* rec, int64_t cap, int64_t* n_out) {
  if (h && h->host_only) return fail(PT_EINVAL, "plan-only handle (PT_DEVICE_HOST)");
  if (!h || !in || !out || !rec || !n_out) return fail(PT_EINVAL, "null argument");
  DeviceGuard guard(h->device);
  const char* names[] = {"A", "M", "AM", "S"};
  if (kind < 0 || kind > 3) return fail(PT_EINVAL, "unknown program kind");
  if (kind != 0 && !h->sweep_err.empty()) return fail(PT_EINVAL, h->sweep_err);
  DevProgram* p;
  int rc = get_program(h, names[kind], kind == 0 || kind == 3 ? 0 : n_it, &p);
  if (rc) return rc;
  const int64_t nt = (int64_t)p->host.tasks.size();
  *n_out = nt;
  if (cap < nt) return fail(PT_EINVAL, "trace buffer too small");
  CK(cudaDeviceSynchronize());
  const size_t words = (size_t)std::max<int64_t>(nt, 1) * EXEC_TRACE;
  CK(cudaMalloc(&h->trace_buf, words * sizeof(unsigned long long)));
  CK(cudaMemset(h->trace_buf, 0, words * sizeof(unsigned long long)));
  rc = run_program(h, p, (const double2*)in, (double2*)out, (const double2*)in, 0);
  std::vector<unsigned long long> tr(words);
  cudaError_t e1 = cudaDeviceSynchronize();
  cudaError_t e2 = cudaMemcpy(tr.data(), h->trace_buf, tr.size() * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost);
  cudaFree(h->trace_buf);
  h->trace_buf = nullptr;
  if (rc) return rc;
  CK(e1);
  CK(e2);
  for (int64_t q = 0; q < nt; ++q) {
    const DevTask& t = p->host.tasks[q];
    const unsigned long long* w = tr.data() + EXEC_TRACE * q;
    int64_t* r = rec + PT_TRACE_WORDS * q;
    r[0] = t.type;
    r[1] = t.out.slot;
    r[2] = t.out.off;
    r[3] = t.r0;
    r[4] = t.r1;
    r[5] = t.nterm;
    r[6] = (int64_t)w[0];   // grabbed
    r[7] = (int64_t)w[1];   // dependencies satisfied
    r[8] = (int64_t)w[2];   // done
    r[9] = (int64_t)w[3];   // SM id | CTA index << 16
    r[10] = (int64_t)w[4];  // consumers started
    r[11] = t.signal;
    r[12] = (int64_t)w[5];  // vectors staged
    r[13] = t.npiece;
    for (int k = 0; k < 8; ++k) {
      r[14 + k] = (int64_t)w[14 + k];  // piece k issued
      r[22 + k] = (int64_t)w[6 + k];   // piece k landed (consumer view)
    }
    r[30] = (int64_t)w[22];  // consumer cycles waiting for pieces
    r[31] = (int64_t)w[23];  // consumer cycles in the per-piece barrier
  }
  return 0;
}

int pt_plan_stats(pt_handle* h, int32_t kind, int32_t n_it, int64_t* stats) {
  if (!h || !stats) return fail(PT_EINVAL, "null argument");
  if (kind < 0 || kind > 3) return fail(PT_EINVAL, "unknown program kind");
  if (kind == 1 || kind == 2) {
    if (n_it < 1) return fail(PT_EINVAL, "n_it must be at least 1");
    if (!h->sweep_err.empty()) return fail(PT_EINVAL, h->sweep_err);
  }
  if (kind == 3 && !h->sweep_err.empty()) return fail(PT_EINVAL, h->sweep_err);
  FusedGeom scope(h, kind == 2);
  Program pg = kind == 0   ? build_apply_A(h->op, h->pp)
               : kind == 1 ? build_apply_M(h->op, n_it, h->pp)
               : kind == 2 ? build_A_then_M(h->op, n_it, h->pp)
                           : build_gs_sweep(h->op, h->pp);
  for (int i = 0; i < PT_PLAN_STATS; ++i) stats[i] = 0;
  stats[0] = (int64_t)pg.tasks.size();
  for (const DevTask& t : pg.tasks) {
    stats[t.type == TASK_T_PLR ? 1 : t.type == TASK_Y_PLR ? 2 : 3] += 1;
    stats[9] = std::max<int64_t>(stats[9], t.nterm);
    stats[10] = std::max<int64_t>(stats[10], t.npiece);
    stats[11] = std::max<int64_t>(stats[11], t.nitem);
  }
  if (int rc = check_slots(h, pg)) return rc;
  {
    std::vector<int4> blob;
    std::vector<int64_t> off;
    int64_t mx = 0;
    build_blobs(pg, blob, off, &mx);
    if (mx > h->blob_cap) return fail(PT_EINVAL, "a task's metadata exceeds the executor's task slot");
  }
  stats[4] = (int64_t)pg.pieces.size();
  stats[5] = (int64_t)pg.items.size();
  stats[6] = pg.n_counters;
  stats[7] = (int64_t)pg.algo_bytes;
  for (const DevPiece& pc : pg.pieces) stats[8] += 16 * (int64_t)(pc.elems + pc.elems2);
  if (!pg.overflow.empty()) return fail(PT_EINVAL, pg.overflow);
  return 0;
}

int pt_plan_tasks(pt_handle* h, int32_t kind, int32_t n_it, int32_t* rec, int64_t cap,
                  int64_t* n_out) {
  if (!h || !rec || !n_out) return fail(PT_EINVAL, "null argument");
  if (kind < 0 || kind > 3) return fail(PT_EINVAL, "unknown program kind");
  if ((kind == 1 || kind == 2) && n_it < 1) return fail(PT_EINVAL, "n_it must be at least 1");
  if (kind != 0 && !h->sweep_err.empty()) return fail(PT_EINVAL, h->sweep_err);
  FusedGeom scope(h, kind == 2);
  Program pg = kind == 0   ? build_apply_A(h->op, h->pp)
               : kind == 1 ? build_apply_M(h->op, n_it, h->pp)
               : kind == 2 ? build_A_then_M(h->op, n_it, h->pp)
                           : build_gs_sweep(h->op, h->pp);
  const int64_t nt = (int64_t)pg.tasks.size();
  *n_out = nt;
  if (cap < nt) return fail(PT_EINVAL, "task record buffer too small");
  for (int64_t q = 0; q < nt; ++q) {
    const DevTask& t = pg.tasks[q];
    int32_t* r = rec + PT_TASK_WORDS * q;
    r[0] = t.type;
    r[1] = t.signal;
    r[2] = t.nwait | ((q < (int64_t)pg.chain.size() && pg.chain[q]) ? 1 << 16 : 0);
    r[3] = t.npiece;
    r[4] = t.r0;
    r[5] = t.r1;
    int64_t elems = 0;  // operator elements the task stages
    for (int32_t i = 0; i < t.npiece; ++i) elems += pg.pieces[t.piece0 + i].elems + pg.pieces[t.piece0 + i].elems2;
    r[6] = t.out.slot | (t.nitem << 8);
    r[7] = (int32_t)elems;
    for (int i = 0; i < 8; ++i) {
      const bool has = i < t.nwait;
      r[8 + 2 * i] = has ? pg.waits[t.wait0 + i].ctr : -1;
      r[9 + 2 * i] = has ? pg.waits[t.wait0 + i].val : 0;
    }
  }
  return 0;
}

int pt_exec_info(const pt_handle* h, int32_t* grid, int64_t* smem_bytes, int64_t* half_elems) {
  if (!h) return fail(PT_EINVAL, "null handle");
  if (grid) *grid = h->grid;
  if (smem_bytes) *smem_bytes = (int64_t)h->smem;
  if (half_elems) *half_elems = h->pp.half_elems;
  return 0;
}

int64_t pt_bytes_apply_A(const pt_handle* hc) {
  pt_handle* h = const_cast<pt_handle*>(hc);
  if (!h) return -1;
  DeviceGuard guard(h->device);
  DevProgram* p;
  if (get_program(h, "A", 0, &p)) return -1;
  return p->host.algo_bytes;
}

int64_t pt_bytes_apply_M(const pt_handle* hc, int32_t n_it) {
  pt_handle* h = const_cast<pt_handle*>(hc);
  if (!h || n_it < 1 || !h->sweep_err.empty()) return -1;
  DeviceGuard guard(h->device);
  DevProgram* p;
  if (get_program(h, "M", n_it, &p)) return -1;
  return p->host.algo_bytes;
}

}  // extern "C"
