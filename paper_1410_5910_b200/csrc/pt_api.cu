// C ABI (include/pt_b200.h): upload, program cache, launches, GMRES driver.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "pt_b200.h"
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

int fail(int code, const std::string& msg) {
  g_err = msg;
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
  ~DevProgram() {
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
  int* nonfinite = nullptr;
  DevStatus* st_host = nullptr;  // pinned
  ~pt_gmres_ws() {
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
    cudaFree(nonfinite);
    cudaFreeHost(st_host);
  }
};

struct pt_handle {
  int device = 0;
  Operator op;
  std::string sweep_err;
  PlanParams pp;
  double2* dense = nullptr;
  double2* fac = nullptr;
  DevLeaf* leaves = nullptr;
  DevSlot* slots = nullptr;
  DevKernelPLR* kplr = nullptr;
  int32_t* rowseg = nullptr;
  DevSegment* segs = nullptr;
  int32_t* seg_leaves = nullptr;
  std::map<std::string, std::unique_ptr<DevProgram>> progs;
  double2* slot_buf[N_SLOTS] = {nullptr};
  int64_t slot_cap[N_SLOTS] = {0};
  int* ctr = nullptr;
  int ctr_cap = 0;
  int grid = 0;
  size_t smem = 0;
  std::unique_ptr<pt_gmres_ws> gws;
  double2* tmp = nullptr;
  double2* hb = nullptr;  // device staging for the *_host solve
  double2* hx = nullptr;
  ~pt_handle() {
    progs.clear();
    cudaFree(dense);
    cudaFree(fac);
    cudaFree(leaves);
    cudaFree(slots);
    cudaFree(kplr);
    cudaFree(rowseg);
    cudaFree(segs);
    cudaFree(seg_leaves);
    for (int s = 0; s < N_SLOTS; ++s) cudaFree(slot_buf[s]);
    cudaFree(ctr);
    cudaFree(tmp);
    cudaFree(hb);
    cudaFree(hx);
  }
  int64_t N() const { return op.nb * op.m; }
};

namespace {

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
  op.kplr.assign(op.nk, DevKernelPLR{});
  op.nslot.assign(op.nk, 0);
  op.kernel_bytes.assign(op.nk, 0);
  op.rowseg.assign((size_t)op.nk * m, 0);
  size_t pos = 0;
  for (int k = 0; k < op.nk; ++k) {
    DevKernelPLR& kp = op.kplr[k];
    kp.leaf0 = (int32_t)op.leaves.size();
    kp.slot0 = (int32_t)op.slots.size();
    int32_t slot = 0;
    std::vector<int64_t> bounds = {0, m};
    for (; pos < idx.size() && leaves[idx[pos]].kernel == k; ++pos) {
      const pt_leaf& L = leaves[idx[pos]];
      op.kernel_bytes[k] += 16 * L.rank * (L.rows + L.cols);
      if (L.rank == 0) continue;
      DevLeaf dl{};
      align8();
      dl.u_off = (int64_t)blob.size();
      const double* U = fac + 2 * L.u_off;
      for (int64_t c = 0; c < L.rank; ++c)
        for (int64_t r = 0; r < L.rows; ++r) {
          const double* z = U + 2 * (r * L.rank + c);
          blob.push_back(make_double2(z[0], z[1]));
        }
      align8();
      dl.v_off = (int64_t)blob.size();
      const double* Vt = fac + 2 * L.vt_off;
      for (int64_t i = 0; i < L.rank * L.cols; ++i) blob.push_back(make_double2(Vt[2 * i], Vt[2 * i + 1]));
      dl.row_off = (int32_t)L.row_off;
      dl.col_off = (int32_t)L.col_off;
      dl.rows = (int32_t)L.rows;
      dl.cols = (int32_t)L.cols;
      dl.rank = (int32_t)L.rank;
      dl.slot0 = slot;
      for (int64_t c = 0; c < L.rank; ++c) {
        DevSlot s{};
        s.v_off = dl.v_off + c * L.cols;
        s.col_off = dl.col_off;
        s.cols = dl.cols;
        op.slots.push_back(s);
      }
      slot += (int32_t)L.rank;
      op.leaves.push_back(dl);
      bounds.push_back(L.row_off);
      bounds.push_back(L.row_off + L.rows);
    }
    kp.nleaf = (int32_t)op.leaves.size() - kp.leaf0;
    kp.nslot = slot;
    op.nslot[k] = slot;
    std::sort(bounds.begin(), bounds.end());
    bounds.erase(std::unique(bounds.begin(), bounds.end()), bounds.end());
    kp.seg0 = (int32_t)(k * m);
    for (size_t b = 0; b + 1 < bounds.size(); ++b) {
      const int64_t lo = bounds[b], hi = bounds[b + 1];
      DevSegment sg{};
      sg.leaf_list0 = (int32_t)op.seg_leaves.size();
      for (int32_t l = kp.leaf0; l < kp.leaf0 + kp.nleaf; ++l) {
        const DevLeaf& dl = op.leaves[l];
        if (dl.row_off <= lo && dl.row_off + dl.rows >= hi) op.seg_leaves.push_back(l);
      }
      sg.nleaf = (int32_t)op.seg_leaves.size() - sg.leaf_list0;
      const int32_t sid = (int32_t)op.segs.size();
      op.segs.push_back(sg);
      for (int64_t r = lo; r < hi; ++r) op.rowseg[(size_t)k * m + r] = sid;
    }
  }
  if (op.seg_leaves.empty()) op.seg_leaves.push_back(0);
  if (blob.empty()) blob.push_back(make_double2(0.0, 0.0));
  int rc;
  if ((rc = upload(&h->fac, blob))) return rc;
  if ((rc = upload(&h->leaves, op.leaves))) return rc;
  if ((rc = upload(&h->slots, op.slots))) return rc;
  if ((rc = upload(&h->kplr, op.kplr))) return rc;
  if ((rc = upload(&h->rowseg, op.rowseg))) return rc;
  if ((rc = upload(&h->segs, op.segs))) return rc;
  if ((rc = upload(&h->seg_leaves, op.seg_leaves))) return rc;
  return 0;
}

int ensure_slot(pt_handle* h, int s, int64_t elems) {
  if (elems <= h->slot_cap[s]) return 0;
  CK(cudaDeviceSynchronize());
  cudaFree(h->slot_buf[s]);
  h->slot_buf[s] = nullptr;
  CK(cudaMalloc(&h->slot_buf[s], (size_t)std::max<int64_t>(elems, 1) * sizeof(double2)));
  CK(cudaMemset(h->slot_buf[s], 0, (size_t)std::max<int64_t>(elems, 1) * sizeof(double2)));
  h->slot_cap[s] = elems;
  return 0;
}

int get_program(pt_handle* h, const std::string& kind, int n_it, DevProgram** out) {
  const std::string key = kind + std::to_string(n_it);
  auto it = h->progs.find(key);
  if (it != h->progs.end()) {
    *out = it->second.get();
    return 0;
  }
  std::unique_ptr<DevProgram> p(new DevProgram());
  if (kind == "A")
    p->host = build_apply_A(h->op, h->pp);
  else if (kind == "M")
    p->host = build_apply_M(h->op, n_it, h->pp);
  else if (kind == "S")
    p->host = build_gs_sweep(h->op, h->pp);
  else
    p->host = build_A_then_M(h->op, n_it, h->pp);
  int rc;
  if ((rc = upload(&p->tasks, p->host.tasks))) return rc;
  if ((rc = upload(&p->terms, p->host.terms))) return rc;
  if ((rc = upload(&p->eyes, p->host.eyes))) return rc;
  if ((rc = upload(&p->waits, p->host.waits))) return rc;
  for (int s : {SLOT_Y, SLOT_U1, SLOT_U2, SLOT_PRE, SLOT_T})
    if ((rc = ensure_slot(h, s, p->host.slot_elems[s]))) return rc;
  if (p->host.n_counters + 1 > h->ctr_cap) {
    CK(cudaDeviceSynchronize());
    cudaFree(h->ctr);
    h->ctr_cap = p->host.n_counters + 1;
    CK(cudaMalloc(&h->ctr, h->ctr_cap * sizeof(int)));
  }
  *out = p.get();
  h->progs[key] = std::move(p);
  return 0;
}

int run_program(pt_handle* h, DevProgram* p, const double2* in, double2* out, const double2* aux,
                cudaStream_t s) {
  if (p->host.tasks.empty()) return 0;
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
  a.rowseg = h->rowseg;
  a.segs = h->segs;
  a.seg_leaves = h->seg_leaves;
  a.n_tasks = (int)p->host.tasks.size();
  a.m = (int)h->op.m;
  CK(cudaMemsetAsync(h->ctr, 0, (p->host.n_counters + 1) * sizeof(int), s));
  void* args[] = {&a};
  count_launch();
  CK(cudaLaunchCooperativeKernel((const void*)pt_exec_kernel, dim3(h->grid), dim3(EXEC_THREADS),
                                 args, h->smem, s));
  return 0;
}

int ws_alloc(pt_gmres_ws* w, int64_t n, int max_iter) {
  GmresDev& d = w->d;
  d.n = n;
  d.max_iter = max_iter;
  d.ldp = max_iter + 2;
  const size_t ldr = (size_t)max_iter + 1;
  CK(cudaMalloc(&d.V, (size_t)n * ldr * sizeof(double2)));
  CK(cudaMalloc(&d.P, (size_t)RED_BLOCKS * d.ldp * sizeof(double2)));
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
  CK(cudaMalloc(&w->nonfinite, sizeof(int)));
  CK(cudaMallocHost(&w->st_host, sizeof(DevStatus)));
  CK(cudaMemset(d.st, 0, sizeof(DevStatus)));
  return 0;
}

int fetch_status(pt_gmres_ws* w, cudaStream_t s) {
  CK(cudaMemcpyAsync(w->st_host, w->d.st, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}

int ws_begin_impl(pt_gmres_ws* w, const double* mb, double* beta_out, cudaStream_t s) {
  GmresDev& d = w->d;
  if ((const double2*)mb != d.V)
    CK(cudaMemcpyAsync(d.V, mb, d.n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  CK(cudaMemsetAsync(w->nonfinite, 0, sizeof(int), s));
  gm_norm(d.V, d.n, d.P, d.ldp, nullptr, s);
  gm_reduce(d.P, d.ldp, 1, d.hn2, s);
  gm_begin(d, s);
  gm_scale(d.V, d.n, d.st, 1, s);
  CK(cudaGetLastError());
  int rc = fetch_status(w, s);
  if (rc) return rc;
  if (beta_out) *beta_out = w->st_host->beta;
  return 0;
}

int ws_step_impl(pt_gmres_ws* w, int j, double rel_tol, int max_iter, pt_report* rep, int* stop,
                 cudaStream_t s) {
  GmresDev& d = w->d;
  if (j < 0 || j >= d.max_iter || max_iter > d.max_iter)
    return fail(PT_EINVAL, "GMRES step index outside the workspace");
  double2* wv = d.V + (int64_t)(j + 1) * d.n;
  const int nc = j + 1;
  gm_dots(d.V, d.n, nc, wv, d.n, d.P, d.ldp, w->nonfinite, s);
  gm_reduce(d.P, d.ldp, nc, d.h1, s);
  gm_update_dots(d.V, d.n, nc, d.h1, wv, d.n, d.P, d.ldp, s);
  gm_reduce(d.P, d.ldp, nc, d.h2, s);
  gm_update_norm(d.V, d.n, nc, d.h2, wv, d.n, d.P, d.ldp, s);
  gm_reduce(d.P, d.ldp, 1, d.hn2, s);
  gm_givens(d, j, rel_tol, max_iter, w->nonfinite, s);
  gm_scale(wv, d.n, d.st, 0, s);
  CK(cudaGetLastError());
  int rc = fetch_status(w, s);
  if (rc) return rc;
  const DevStatus& st = *w->st_host;
  if (st.nonfinite) {
    if (rep) rep->nonfinite = 1;
    return fail(PT_ENONFINITE, "non-finite values in preconditioned matvec at iteration " +
                                   std::to_string(j + 1));
  }
  if (rep) {
    rep->iterations = st.iterations;
    rep->flag = st.flag;
    rep->converged = st.converged;
    rep->beta = st.beta;
    if (rep->residual_history) rep->residual_history[j] = st.rel;
  }
  *stop = st.stop;
  return 0;
}

int ensure_gws(pt_handle* h, int max_iter) {
  if (h->gws && h->gws->d.max_iter >= max_iter) return 0;
  CK(cudaDeviceSynchronize());
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

int pt_create(const pt_layout* layout, const pt_entry* entries, int64_t n_entries,
              const int64_t* perm, const double* dense, const pt_leaf* leaves, int64_t n_leaves,
              const double* factors, int64_t n_factor_complex, int device, pt_handle** out) {
  if (!layout || !out || (n_entries > 0 && !entries) || !perm)
    return fail(PT_EINVAL, "null argument to pt_create");
  *out = nullptr;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(PT_EINVAL, "no such CUDA device");
  DeviceGuard guard(device);
  std::unique_ptr<pt_handle> h(new pt_handle());
  h->device = device;
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
  if (op.fmt == PT_KERNEL_DENSE) {
    op.kernel_bytes.assign(op.nk, 16 * op.m * op.m);
    if (op.nk > 0) {
      if (!dense) return fail(PT_EINVAL, "dense kernel array missing");
      const size_t bytes = (size_t)op.nk * op.m * op.m * sizeof(double2);
      CK(cudaMalloc(&h->dense, bytes));
      CK(cudaMemcpy(h->dense, dense, bytes, cudaMemcpyHostToDevice));
    }
  } else {
    if (n_leaves > 0 && (!leaves || !factors)) return fail(PT_EINVAL, "PLR tables missing");
    if ((rc = build_plr_tables(h.get(), leaves, n_leaves, factors, n_factor_complex))) return rc;
  }
  h->smem = (size_t)op.m * sizeof(double2);
  if (h->smem > 48 * 1024)
    CK(cudaFuncSetAttribute(pt_exec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)h->smem));
  int nsm = 0, occ = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pt_exec_kernel, EXEC_THREADS, h->smem));
  if (occ < 1) return fail(PT_EINVAL, "executor kernel does not fit on an SM");
  h->grid = nsm * occ;
  h->pp.dense_rows_per_task = DENSE_ROWS_PER_TASK;
  h->pp.plr_rows_per_task = EXEC_THREADS;
  CK(cudaMalloc(&h->tmp, std::max<int64_t>(h->N(), 1) * sizeof(double2)));
  *out = h.release();
  return 0;
}

int pt_destroy(pt_handle* h) {
  if (!h) return 0;
  DeviceGuard guard(h->device);
  cudaDeviceSynchronize();
  delete h;
  return 0;
}

int pt_apply_A(pt_handle* h, const double* x, double* y, pt_stream stream) {
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

int pt_gs_sweep(pt_handle* h, const double* rhs, const double* u_in, double* u_out,
                pt_stream stream) {
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

int pt_gmres(pt_handle* h, const double* b, double* x, const pt_gmres_config* cfg,
             pt_report* report, pt_stream stream) {
  if (!h || !b || !x) return fail(PT_EINVAL, "null argument");
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (!h->sweep_err.empty()) return fail(PT_EINVAL, h->sweep_err);
  DeviceGuard guard(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  if ((rc = ensure_gws(h, cfg->max_iter))) return rc;
  pt_gmres_ws* w = h->gws.get();
  GmresDev& d = w->d;
  DevProgram *pM, *pAM, *pA;
  if ((rc = get_program(h, "M", cfg->n_it, &pM))) return rc;
  if ((rc = get_program(h, "AM", cfg->n_it, &pAM))) return rc;
  if ((rc = get_program(h, "A", 0, &pA))) return rc;
  pt_report local{};
  pt_report* rep = report ? report : &local;
  double* hist = rep->residual_history;
  *rep = pt_report{};
  rep->residual_history = hist;
  rep->flag = PT_FLAG_CONVERGED;
  const int64_t N = h->N();
  // mb = M^-1 b straight into basis column 0
  if ((rc = run_program(h, pM, (const double2*)b, d.V, nullptr, s))) return rc;
  double beta = 0.0;
  if ((rc = ws_begin_impl(w, (const double*)d.V, &beta, s))) return rc;
  rep->beta = beta;
  if (beta == 0.0) {
    gm_zero((double2*)x, N, s);
    CK(cudaStreamSynchronize(s));
    rep->converged = 1;
    rep->true_residual = 0.0;
    return 0;
  }
  int stop = 0;
  for (int j = 0; j < cfg->max_iter && !stop; ++j) {
    if ((rc = run_program(h, pAM, d.V + (int64_t)j * N, d.V + (int64_t)(j + 1) * N, nullptr, s)))
      return rc;
    if ((rc = ws_step_impl(w, j, cfg->rel_tol, cfg->max_iter, rep, &stop, s))) return rc;
  }
  const int k = rep->iterations;
  gm_backsolve(d, k, s);
  gm_combine(d.V, N, k, d.y, (double2*)x, N, s);
  if ((rc = run_program(h, pA, (const double2*)x, h->tmp, nullptr, s))) return rc;
  gm_resid((const double2*)b, h->tmp, N, d.P, d.ldp, s);
  gm_resid_finish(d, s);
  CK(cudaGetLastError());
  if ((rc = fetch_status(w, s))) return rc;
  const double tr = std::sqrt(w->st_host->true_num2), sc = std::sqrt(w->st_host->b_norm2);
  rep->true_residual = sc > 0.0 ? tr / sc : tr;
  return 0;
}

int pt_gmres_host(pt_handle* h, const double* b_host, double* x_host, const pt_gmres_config* cfg,
                  pt_report* report, pt_stream stream) {
  if (!h || !b_host || !x_host) return fail(PT_EINVAL, "null argument");
  DeviceGuard guard(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = (size_t)h->N() * sizeof(double2);
  if (!h->hb) CK(cudaMalloc(&h->hb, bytes));
  if (!h->hx) CK(cudaMalloc(&h->hx, bytes));
  CK(cudaMemcpyAsync(h->hb, b_host, bytes, cudaMemcpyHostToDevice, s));
  int rc = pt_gmres(h, (const double*)h->hb, (double*)h->hx, cfg, report, stream);
  if (rc) return rc;
  CK(cudaMemcpyAsync(x_host, h->hx, bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}

int pt_gmres_batch(pt_handle* h, const double* b, double* x, int32_t nrhs,
                   const pt_gmres_config* cfg, pt_report* reports, pt_stream stream) {
  if (!h || !b || !x || nrhs < 0) return fail(PT_EINVAL, "bad argument");
  const int64_t N = h->N();
  for (int32_t r = 0; r < nrhs; ++r) {
    int rc = pt_gmres(h, b + 2 * r * N, x + 2 * r * N, cfg, reports ? reports + r : nullptr, stream);
    if (rc) return rc;
  }
  return 0;
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
  return ws_begin_impl(ws, mb, beta_out, (cudaStream_t)stream);
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
  gm_backsolve(ws->d, k, s);
  gm_combine(ws->d.V, ws->d.n, k, ws->d.y, (double2*)x, ws->d.n, s);
  CK(cudaGetLastError());
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
