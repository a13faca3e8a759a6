// Per-layer local solves on the device: Newton traces and volume
// reconstruction.
//
// The reference solves every layer's sparse system with SuperLU on the host
// (LocalFactorization.solve, local_solver.py:21-60) twice per source: once for
// the Newton traces (newton_trace, :138-144) and once for the volume
// (reconstruct_volume, :147-176).  Here the host offline stage factors each
// layer once (offline/local.py: geometric nested-dissection order, SuperLU
// with that order), and the device keeps L and U of ALL layers resident and
// solves them together:
//
//   y = b[q_in]   (the layer's right-hand side, gathered through the composed
//                  row / nested-dissection permutation)
//   L w = y, U z = w   (sparse triangular solves)
//   x = z[q_out]  (back to the layer's natural (z, x) grid order)
//
// Triangular solves are "sync-free": one warp per row, rows handed out from a
// queue sorted by dependency level across all layers (so the layers advance
// together), each warp spins on the flags of the rows its row depends on and
// publishes its own value with a release flag.  One launch per triangular
// factor for every layer; no grid barrier.  Flags carry an epoch, so no reset
// between solves.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "pt_b200.h"
#include "pt_device.cuh"

namespace pt {
extern void count_launch();
}
using namespace pt;

namespace {

thread_local std::string g_lerr;
int lfail(int code, const std::string& m) {
  g_lerr = m;
  return code;
}
#define LCK(x)                                                                          \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) return lfail(PT_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct LayerDev {
  int64_t row0;     // first global row of the layer's unknowns
  int64_t dim;      // nze * nxe
  int32_t nze, nxe, n_layer, n_pml;
  int64_t f_row0;   // extended-grid row of the layer's depth 1
  int64_t u_row0;   // first interior row of the layer in the volume output
  int32_t has_top, has_bot;  // interface above (l >= 2) / below (l <= L-1)
  int32_t top, bot;          // trace blocks 2(l-2) and 2(l-1)
};

// ---- sync-free sparse triangular solve (one warp per row) -------------------
__global__ void __launch_bounds__(1024)
k_trsv(const int* __restrict__ order, int n, const int64_t* __restrict__ ptr,
       const int* __restrict__ col, const double2* __restrict__ val, const double2* __restrict__ dinv,
       const double2* b, double2* x, int* flag, int epoch, int* head, int spin_ns, int chunk) {
  const int lane = threadIdx.x & 31;
  int q = 0, qend = 0;
  for (;;) {
    // `chunk` consecutive queue positions per grab (fewer same-address atomics)
    if (q >= qend) {
      if (lane == 0) q = atomicAdd(head, chunk);
      q = __shfl_sync(0xffffffffu, q, 0);
      qend = min(q + chunk, n);
    }
    if (q >= n) return;
    const int i = __ldg(order + q++);
    const int64_t e0 = __ldg(ptr + i), e1 = __ldg(ptr + i + 1);
    // the row's own data (factor entries, rhs, 1/diagonal) is loaded before
    // any dependency wait, so only the x loads follow a satisfied flag
    // (a warp-per-separator variant that kept dense separator runs in shared
    // memory serialised these loads and measured 2.2x slower)
    const double2 bi = lane == 0 ? ld_cg(b + i) : make_double2(0.0, 0.0);
    const double2 di = lane == 0 ? __ldg(dinv + i) : make_double2(0.0, 0.0);
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const int j = __ldg(col + e);
      const double2 v = __ldg(val + e);
      while (ld_acquire(flag + j) != epoch)
        if (spin_ns) __nanosleep(spin_ns);
      acc = cfma(v, ld_cg(x + j), acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      st_cg(x + i, cmul(csub(bi, acc), di));
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag + i), "r"(epoch) : "memory");
    }
  }
}

// ---- block triangular solve (one CTA per nested-dissection block) ----------
// The factor order is the nested-dissection order, so every leaf block and
// separator is a contiguous run of rows whose diagonal block L_SS (U_SS) is
// triangular and dense enough to invert once at create time.  A block's solve
// is then two parallel steps: r = b_S - L_S,ext x_ext (the entries outside the
// block), x_S = L_SS^-1 r (a dense product) -- instead of one flag round trip
// per row of the block.  Blocks are queued by their dependency level (the
// depth of the dissection tree) and a block waits, once, for every block of
// the lower levels: a done counter reaching qwait[q] (the number of blocks
// queued before q's level).  Completions arrive level by level (a block
// starts only after all lower levels are done), so the count is exact.  The
// off-block product then issues all its loads at once, where a flag check
// per entry cost two dependent L2 round trips per entry.
constexpr int TRSV_BLOCK_MAX = 256;
#ifndef PT_TRSV_THREADS
#define PT_TRSV_THREADS 256
#endif
// threads per block solve (c3 Newton solve: 64 / 128 / 256 / 512 / 1024
// threads 9.8 / 6.6 / 5.5-6.0 / 7.0 / 17.4 ms -- the many small blocks of the
// lower levels want many resident CTAs)
constexpr int TRSV_BLOCK_THREADS = PT_TRSV_THREADS;
__global__ void __launch_bounds__(TRSV_BLOCK_THREADS)
k_trsv_block(const int* __restrict__ border, const int* __restrict__ qwait,
             const int* __restrict__ bstart, const int* __restrict__ blen,
             const int64_t* __restrict__ boff, const double2* __restrict__ binv, int nblocks,
             const int64_t* __restrict__ ptr, const int* __restrict__ col,
             const double2* __restrict__ val, const double2* b, double2* x, int* head, int* done,
             int spin_ns) {
  __shared__ double2 r[TRSV_BLOCK_MAX];
  __shared__ int s_q;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) {
      const int q = atomicAdd(head, 1);
      if (q < nblocks) {
        const int need = __ldg(qwait + q);
        while (ld_acquire(done) < need)
          if (spin_ns) __nanosleep(spin_ns);
      }
      s_q = q;
    }
    __syncthreads();
    const int q = s_q;
    if (q >= nblocks) return;
    const int blk = __ldg(border + q);
    const int s0 = __ldg(bstart + blk), len = __ldg(blen + blk);
    // r = b_S - (entries outside the block) . x   (x of lower levels: final)
    for (int k = wid; k < len; k += nw) {
      const int i = s0 + k;
      const int64_t e0 = __ldg(ptr + i), e1 = __ldg(ptr + i + 1);
      double2 acc = make_double2(0.0, 0.0);
      // four entries per lane in flight (lane order kept: e, e + 32, ...);
      // entries inside the block are left to the inverse
      for (int64_t e = e0 + lane; e < e1; e += 128) {
        int j[4];
        double2 v[4], xv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t f = e + 32 * u;
          j[u] = f < e1 ? __ldg(col + f) : s0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool out = j[u] < s0 || j[u] >= s0 + len;
          v[u] = out ? __ldg(val + e + 32 * u) : make_double2(0.0, 0.0);
          xv[u] = out ? ld_cg(x + j[u]) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (j[u] < s0 || j[u] >= s0 + len) acc = cfma(v[u], xv[u], acc);
      }
      acc = warp_sum(acc);
      if (lane == 0) r[k] = csub(ld_cg(b + i), acc);
    }
    __syncthreads();
    // x_S = inv(L_SS) r (row k of the inverse is contiguous)
    const double2* inv = binv + __ldg(boff + blk);
    for (int k = wid; k < len; k += nw) {
      double2 acc = make_double2(0.0, 0.0);
      for (int j = lane; j < len; j += 32) acc = cfma(__ldg(inv + (int64_t)k * len + j), r[j], acc);
      acc = warp_sum(acc);
      if (lane == 0) st_cg(x + s0 + k, acc);
    }
    __syncthreads();  // r is reused by the next block; x_S written
    if (threadIdx.x == 0)  // release: the block's x_S before the count
      asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(done) : "memory");
  }
}

// Lower levels (every block of the level at most 32 rows: the dissection
// leaves and short separators, ~all of the blocks): one WARP per block, lane k
// owns row k.  Warps grab chunks of TRSV_WARP_CHUNK consecutive queue entries
// (level order) from a queue head, so a block waited on was always grabbed by
// a running warp (no residency assumption), and count their solved blocks
// per level into the level's done counter, flushing before any wait.  A block
// of level l waits for level l - 1's counter to be complete (levels complete
// in order).  Per block: r_k = b_k - (off-block entries of row k) . x, then
// x_k = sum_j inv[k, j] r_j with r_j broadcast by shuffles.
constexpr int TRSV_WARP_MAX = 32;
constexpr int TRSV_WARP_CHUNK = 8;
__global__ void __launch_bounds__(256)
k_trsv_warp(const int* __restrict__ border, const int* __restrict__ qlev,
            const int* __restrict__ lq0, int nq, const int* __restrict__ bstart,
            const int* __restrict__ blen, const int64_t* __restrict__ boff,
            const double2* __restrict__ binv, const int64_t* __restrict__ ptr,
            const int* __restrict__ col, const double2* __restrict__ val, const double2* b,
            double2* x, int* lvl_done, int* whead, int spin_ns) {
  const int lane = threadIdx.x & 31;
  int known = 0;     // levels below this one are known complete
  int pend_l = -1;   // level of the solved blocks not yet counted
  int pend_n = 0;
  auto flush = [&]() {
    __syncwarp();  // every lane's x stores before the release
    if (lane == 0 && pend_n > 0)
      asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(lvl_done + pend_l), "r"(pend_n)
                   : "memory");
    pend_n = 0;
  };
  for (;;) {
    int q0 = 0;
    if (lane == 0) q0 = atomicAdd(whead, TRSV_WARP_CHUNK);
    q0 = __shfl_sync(0xffffffffu, q0, 0);
    if (q0 >= nq) break;
    const int q1 = min(q0 + TRSV_WARP_CHUNK, nq);
    for (int q = q0; q < q1; ++q) {
      const int l = __ldg(qlev + q);
      if (l != pend_l) {
        flush();
        pend_l = l;
      }
      if (l > known) {  // wait for level l - 1 (and so every lower level)
        flush();
        const int need = __ldg(lq0 + l) - __ldg(lq0 + l - 1);
        if (lane == 0)
          while (ld_acquire(lvl_done + l - 1) < need)
            if (spin_ns) __nanosleep(spin_ns);
        __syncwarp();
        known = l;
      }
      const int blk = __ldg(border + q);
      const int s0 = __ldg(bstart + blk), len = __ldg(blen + blk);
      double2 r = make_double2(0.0, 0.0);
      if (lane < len) {
        const int i = s0 + lane;
        const int64_t e0 = __ldg(ptr + i), e1 = __ldg(ptr + i + 1);
        double2 acc = make_double2(0.0, 0.0);
        for (int64_t e = e0; e < e1; ++e) {
          const int j = __ldg(col + e);
          if (j < s0 || j >= s0 + len) acc = cfma(__ldg(val + e), ld_cg(x + j), acc);
        }
        r = csub(ld_cg(b + i), acc);
      }
      const double2* inv = binv + __ldg(boff + blk) + (int64_t)lane * len;
      double2 acc = make_double2(0.0, 0.0);
      for (int jj = 0; jj < len; ++jj) {
        const double2 rj = make_double2(__shfl_sync(0xffffffffu, r.x, jj),
                                        __shfl_sync(0xffffffffu, r.y, jj));
        if (lane < len) acc = cfma(__ldg(inv + jj), rj, acc);
      }
      if (lane < len) st_cg(x + s0 + lane, acc);
      ++pend_n;
    }
  }
  flush();
}

// y[G] = b_layer[q_in[k]] for every global row G = row0 + k.  b_layer is the
// layer's forcing in natural (z, x) order: f restricted to the layer rows
// (restrict_source, partition.py:104-113) plus, when x_traces is given, the
// interface forcing of reconstruct_volume (local_solver.py:160-173) from the
// GMRES solution x (traces = x_down + x_up, block order a_1, b_1, ...).
__global__ void k_gather_rhs(const LayerDev* __restrict__ lay, int n_layers, const int64_t* q_in,
                             int64_t total, const double2* f, const double2* xsol, int64_t nt_m,
                             double w, double2* y) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    int l = 0;
    while (l + 1 < n_layers && lay[l + 1].row0 <= g) ++l;
    const LayerDev& L = lay[l];
    const int64_t idx = q_in[g];
    const int r = (int)(idx / L.nxe), c = (int)(idx % L.nxe);
    double2 v = make_double2(0.0, 0.0);
    if (r >= L.n_pml && r < L.n_pml + L.n_layer) v = f[(L.f_row0 + r - L.n_pml) * L.nxe + c];
    if (xsol) {
      auto tr = [&](int blk) {  // trace block blk, column c
        const int64_t o = (int64_t)blk * L.nxe + c;
        return cadd(xsol[o], xsol[nt_m + o]);
      };
      const int d0 = L.n_pml - 1, d1 = L.n_pml, dn = L.n_pml + L.n_layer - 1, dn1 = L.n_pml + L.n_layer;
      if (L.has_top) {
        if (r == d1) v = cadd(v, make_double2(w * tr(L.top).x, w * tr(L.top).y));           // + w u0
        if (r == d0) v = csub(v, make_double2(w * tr(L.top + 1).x, w * tr(L.top + 1).y));   // - w u1
      }
      if (L.has_bot) {
        if (r == dn1) v = csub(v, make_double2(w * tr(L.bot).x, w * tr(L.bot).y));         // - w un
        if (r == dn) v = cadd(v, make_double2(w * tr(L.bot + 1).x, w * tr(L.bot + 1).y));  // + w un1
      }
    }
    y[g] = v;
  }
}

// Newton traces: out[l][d][c] = x_l at local depth (0, 1, n, n+1)[d], column c
__global__ void k_newton_out(const LayerDev* __restrict__ lay, int n_layers, const int64_t* q_out,
                             const double2* z, double2* out) {
  const int l = blockIdx.y, d = blockIdx.z;
  const LayerDev& L = lay[l];
  const int depth = d == 0 ? 0 : d == 1 ? 1 : d == 2 ? L.n_layer : L.n_layer + 1;
  const int r = L.n_pml + depth - 1;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < L.nxe; c += gridDim.x * blockDim.x)
    out[((int64_t)l * 4 + d) * L.nxe + c] = z[L.row0 + q_out[L.row0 + (int64_t)r * L.nxe + c]];
}

// polarized rhs (trace_system.py:475-484) from the Newton traces:
// top = -[N^i(n_i), N^{i+1}(1)]_i, bottom = -[N^i(n_i + 1), N^{i+1}(0)]_i (jump)
// or 0 (extrapolation)
__global__ void k_polarized_rhs(const double2* nw, int n_layers, int nxe, int64_t nt_m, int jump,
                                double2* rhs) {
  const int64_t total = 2 * nt_m;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const bool bottom = e >= nt_m;
    const int64_t o = bottom ? e - nt_m : e;
    const int blk = (int)(o / nxe), c = (int)(o % nxe);
    const int i = blk / 2 + 1;  // interface 1..L-1
    double2 v = make_double2(0.0, 0.0);
    if (!bottom || jump) {
      // block 2(i-1): layer i at depth n (top) / n+1 (bottom): slots 2 / 3
      // block 2i-1:   layer i+1 at depth 1 (top) / 0 (bottom): slots 1 / 0
      const int l = (blk % 2 == 0) ? i - 1 : i;
      const int slot = (blk % 2 == 0) ? (bottom ? 3 : 2) : (bottom ? 0 : 1);
      const double2 u = nw[((int64_t)l * 4 + slot) * nxe + c];
      v = make_double2(-u.x, -u.y);
    }
    rhs[e] = v;
  }
}

// volume: u[(u_row0 + r) * nxe + c] = x_l at layer row n_pml + r, r < n_layer
__global__ void k_volume_out(const LayerDev* __restrict__ lay, int n_layers, const int64_t* q_out,
                             const double2* z, double2* u) {
  const int l = blockIdx.y;
  const LayerDev& L = lay[l];
  const int64_t n = (int64_t)L.n_layer * L.nxe;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / L.nxe, c = e % L.nxe;
    u[(L.u_row0 + r) * L.nxe + c] = z[L.row0 + q_out[L.row0 + (L.n_pml + r) * L.nxe + c]];
  }
}

// dst[g] = src[row0(layer of g) + q[g]]  (q layer-local)
__global__ void k_gather(const int64_t* __restrict__ q, const LayerDev* __restrict__ lay, int nl,
                         int64_t n, const double2* src, double2* dst) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x) {
    int l = 0;
    while (l + 1 < nl && lay[l + 1].row0 <= g) ++l;
    dst[g] = src[lay[l].row0 + q[g]];
  }
}

int elem_grid(int64_t n) { return (int)std::min<int64_t>(std::max<int64_t>((n + 255) / 256, 1), 4096); }

}  // namespace

struct pt_local {
  int device = 0;
  int n_layers = 0;
  int64_t rows = 0;   // total unknowns over the layers
  int64_t nz = 0;     // interior rows of the volume
  int64_t nxe = 0;
  std::vector<LayerDev> host_layers;
  LayerDev* layers = nullptr;
  // factors (global row / column indices), off-diagonal CSR + 1/diagonal
  int64_t *l_ptr = nullptr, *u_ptr = nullptr;
  int *l_col = nullptr, *u_col = nullptr;
  double2 *l_val = nullptr, *u_val = nullptr, *l_dinv = nullptr, *u_dinv = nullptr;
  int *l_order = nullptr, *u_order = nullptr;
  int64_t *q_in = nullptr, *q_out = nullptr;
  double2 *y = nullptr, *w = nullptr, *z = nullptr;
  double2* newton = nullptr;  // Newton traces scratch (n_layers x 4 x nxe)
  int* flag = nullptr;  // [rows] for L, [rows] for U
  int* head = nullptr;  // queue heads and block done counters (2 + 2 per solve)
  int epoch = 0;
  int grid = 0;
  int spin_ns = 0;  // back-off of a warp waiting on a dependency (PT_TRSV_SPIN)
  int chunk = 2;    // queue positions per grab (PT_TRSV_CHUNK; 2 measured best)
  int64_t factor_nnz = 0;
  int32_t l_levels = 0, u_levels = 0;
  // block solve (k_trsv_block): blocks, their inverses, queues by level
  bool blocked = false;  // every layer passed its dissection blocks (PT_TRSV_BLOCK=0: off)
  int nblocks = 0;
  int *bstart = nullptr, *blen = nullptr, *l_border = nullptr, *u_border = nullptr;
  int *l_qwait = nullptr, *u_qwait = nullptr;  // per queue index: blocks of lower levels
  // warp-per-block prefix of each queue (levels whose blocks all have <= 32
  // rows): level starts lq0[0..nlev], queue split
  int *l_lq0 = nullptr, *u_lq0 = nullptr, *l_qlev = nullptr, *u_qlev = nullptr;
  int l_wlev = 0, u_wlev = 0, l_split = 0, u_split = 0;
  int wgrid = 0;
  int64_t *l_boff = nullptr, *u_boff = nullptr;
  double2 *l_binv = nullptr, *u_binv = nullptr;
  int bgrid = 0;
  int32_t l_blevels = 0, u_blevels = 0;
  ~pt_local() {
    for (void* p : {(void*)layers, (void*)l_ptr, (void*)u_ptr, (void*)l_col, (void*)u_col,
                    (void*)l_val, (void*)u_val, (void*)l_dinv, (void*)u_dinv, (void*)l_order,
                    (void*)u_order, (void*)q_in, (void*)q_out, (void*)y, (void*)w, (void*)z, (void*)newton,
                    (void*)flag, (void*)head, (void*)bstart, (void*)blen, (void*)l_border,
                    (void*)u_border, (void*)l_qwait, (void*)u_qwait, (void*)l_lq0, (void*)u_lq0, (void*)l_qlev, (void*)u_qlev,
                    (void*)l_boff, (void*)u_boff,
                    (void*)l_binv, (void*)u_binv})
      cudaFree(p);
  }
};

namespace {

template <class T>
int up(T** dst, const std::vector<T>& v) {
  *dst = nullptr;
  if (v.empty()) return 0;
  LCK(cudaMalloc((void**)dst, v.size() * sizeof(T)));
  LCK(cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return 0;
}

// Split one layer's CSR factor (rows of the permuted system, complex values)
// into off-diagonal entries (global columns) and 1/diagonal; dependency
// levels (lower: rows ascending; upper: descending).
int split_factor(const int64_t* ptr, const int32_t* col, const double* val, int64_t dim,
                 int64_t row0, bool lower, std::vector<int64_t>& gptr, std::vector<int>& gcol,
                 std::vector<double2>& gval, std::vector<double2>& dinv, std::vector<int>& level) {
  std::vector<int> lv(dim, 0);
  std::vector<double2> d(dim, make_double2(0.0, 0.0));
  std::vector<char> has(dim, 0);
  // off-diagonals (and levels, which need rows in dependency order)
  const int64_t base = (int64_t)gcol.size();
  (void)base;
  for (int64_t r = 0; r < dim; ++r) {
    for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) {
      const int64_t c = col[e];
      if (c < 0 || c >= dim) return lfail(PT_EINVAL, "local factor column out of range");
      if (c == r) {
        d[r] = make_double2(val[2 * e], val[2 * e + 1]);
        has[r] = 1;
      } else if ((c < r) != lower) {
        return lfail(PT_EINVAL, lower ? "L factor has entries above the diagonal"
                                      : "U factor has entries below the diagonal");
      }
    }
  }
  for (int64_t k = 0; k < dim; ++k) {
    const int64_t r = lower ? k : dim - 1 - k;
    int m = 0;
    for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e)
      if (col[e] != r) m = std::max(m, lv[col[e]] + 1);
    lv[r] = m;
  }
  for (int64_t r = 0; r < dim; ++r) {
    if (!has[r] || (d[r].x == 0.0 && d[r].y == 0.0))
      return lfail(PT_EINVAL, "local factor has a zero or missing diagonal");
    const double dd = d[r].x * d[r].x + d[r].y * d[r].y;
    dinv.push_back(make_double2(d[r].x / dd, -d[r].y / dd));
    for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e)
      if (col[e] != r) {
        gcol.push_back((int)(row0 + col[e]));
        gval.push_back(make_double2(val[2 * e], val[2 * e + 1]));
      }
    gptr.push_back((int64_t)gcol.size());
    level.push_back(lv[r]);
  }
  return 0;
}

std::vector<int> level_order(const std::vector<int>& level, int32_t* nlev) {
  const int n = (int)level.size();
  int mx = 0;
  for (int v : level) mx = std::max(mx, v);
  *nlev = mx + 1;
  std::vector<int> cnt(mx + 2, 0), order(n);
  for (int v : level) cnt[v + 1]++;
  for (int v = 0; v <= mx; ++v) cnt[v + 1] += cnt[v];
  for (int i = 0; i < n; ++i) order[cnt[level[i]]++] = i;  // stable: layers interleave per level
  return order;
}

// Inverse of the dense diagonal block rows/cols [s0, s0 + n) of one factor
// (off-diagonal CSR with global columns + 1/diagonal), row-major, appended
// to inv.  Lower: forward substitution per column; upper: backward.
void invert_block(const std::vector<int64_t>& ptr, const std::vector<int>& col,
                  const std::vector<double2>& val, const std::vector<double2>& dinv, int64_t s0,
                  int n, bool lower, std::vector<double2>& inv) {
  std::vector<double2> D((size_t)n * n, make_double2(0.0, 0.0));  // strict part
  for (int k = 0; k < n; ++k)
    for (int64_t e = ptr[s0 + k]; e < ptr[s0 + k + 1]; ++e) {
      const int64_t j = col[e] - s0;
      if (j >= 0 && j < n) D[(size_t)k * n + j] = val[e];
    }
  const size_t base = inv.size();
  inv.resize(base + (size_t)n * n, make_double2(0.0, 0.0));
  double2* X = inv.data() + base;
  auto mul = [](double2 a, double2 b2) {
    return make_double2(a.x * b2.x - a.y * b2.y, a.x * b2.y + a.y * b2.x);
  };
  for (int c = 0; c < n; ++c) {
    // column c of the inverse: T x = e_c
    if (lower) {
      for (int k = c; k < n; ++k) {
        double2 acc = make_double2(k == c ? 1.0 : 0.0, 0.0);
        for (int j = c; j < k; ++j) {
          const double2 t = mul(D[(size_t)k * n + j], X[(size_t)j * n + c]);
          acc.x -= t.x;
          acc.y -= t.y;
        }
        X[(size_t)k * n + c] = mul(acc, dinv[s0 + k]);
      }
    } else {
      for (int k = c; k >= 0; --k) {
        double2 acc = make_double2(k == c ? 1.0 : 0.0, 0.0);
        for (int j = k + 1; j <= c; ++j) {
          const double2 t = mul(D[(size_t)k * n + j], X[(size_t)j * n + c]);
          acc.x -= t.x;
          acc.y -= t.y;
        }
        X[(size_t)k * n + c] = mul(acc, dinv[s0 + k]);
      }
    }
  }
}

// queue of blocks by dependency level (lower: deps on earlier blocks;
// upper: on later ones), and the level count
std::vector<int> block_queue(const std::vector<int64_t>& ptr, const std::vector<int>& col,
                             const std::vector<int>& bstart, const std::vector<int>& blen,
                             const std::vector<int>& bid, bool lower, int32_t* nlev,
                             std::vector<int>& qwait) {
  const int nb = (int)bstart.size();
  std::vector<int> lev(nb, 0);
  for (int t = 0; t < nb; ++t) {
    const int b2 = lower ? t : nb - 1 - t;
    int lv = 0;
    for (int64_t i = bstart[b2]; i < bstart[b2] + blen[b2]; ++i)
      for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) {
        const int o = bid[col[e]];
        if (o != b2) lv = std::max(lv, lev[o] + 1);
      }
    lev[b2] = lv;
  }
  std::vector<int> order = level_order(lev, nlev);
  // qwait[q]: blocks queued at lower levels than queue entry q's
  std::vector<int> below(*nlev + 1, 0);
  for (int v : lev) below[v + 1]++;
  for (int v = 0; v < *nlev; ++v) below[v + 1] += below[v];
  qwait.resize(nb);
  for (int q = 0; q < nb; ++q) qwait[q] = below[lev[order[q]]];
  return order;
}

int trsv(pt_local* h, bool lower, const double2* b, double2* x, cudaStream_t s) {
  const int e = h->epoch;
  if (h->blocked) {
    const int split = lower ? h->l_split : h->u_split;
    const int* border = lower ? h->l_border : h->u_border;
    if (split > 0) {  // small lower levels: a warp per block
      k_trsv_warp<<<h->wgrid, 256, 0, s>>>(
          border, lower ? h->l_qlev : h->u_qlev, lower ? h->l_lq0 : h->u_lq0, split, h->bstart,
          h->blen, lower ? h->l_boff : h->u_boff, lower ? h->l_binv : h->u_binv,
          lower ? h->l_ptr : h->u_ptr, lower ? h->l_col : h->u_col, lower ? h->l_val : h->u_val, b,
          x, h->head + (lower ? 4 : 4 + 32), h->head + (lower ? 68 : 69), h->spin_ns);
      LCK(cudaGetLastError());
      count_launch();
    }
    if (split < h->nblocks) {
      count_launch();  // the rest: a CTA per block (qwait counts past the split)
      k_trsv_block<<<h->bgrid, TRSV_BLOCK_THREADS, 0, s>>>(
          border + split, (lower ? h->l_qwait : h->u_qwait) + split, h->bstart, h->blen,
          lower ? h->l_boff : h->u_boff, lower ? h->l_binv : h->u_binv, h->nblocks - split,
          lower ? h->l_ptr : h->u_ptr, lower ? h->l_col : h->u_col, lower ? h->l_val : h->u_val, b,
          x, h->head + (lower ? 0 : 1), h->head + (lower ? 2 : 3), h->spin_ns);
      LCK(cudaGetLastError());
    }
    return 0;
  }
  count_launch();
  k_trsv<<<h->grid, 1024, 0, s>>>(lower ? h->l_order : h->u_order, (int)h->rows,
                                  lower ? h->l_ptr : h->u_ptr, lower ? h->l_col : h->u_col,
                                  lower ? h->l_val : h->u_val, lower ? h->l_dinv : h->u_dinv, b, x,
                                  h->flag + (lower ? 0 : h->rows), e, h->head + (lower ? 0 : 1),
                                  h->spin_ns, h->chunk);
  LCK(cudaGetLastError());
  return 0;
}

// b -> z for every layer: L w = y (y gathered by the caller), U z = w
int solve_all(pt_local* h, cudaStream_t s) {
  ++h->epoch;
  // queue heads, done counters, per-level done counters and queue heads of
  // the warp prefix
  LCK(cudaMemsetAsync(h->head, 0, (4 + 64 + 2) * sizeof(int), s));
  int rc;
  if ((rc = trsv(h, true, h->y, h->w, s))) return rc;
  return trsv(h, false, h->w, h->z, s);
}

}  // namespace

extern "C" {

const char* pt_local_last_error(void) { return g_lerr.c_str(); }

int pt_local_create(const pt_local_layer* layers, int32_t n_layers, int device, pt_local** out) {
  if (!layers || n_layers < 1 || !out) return lfail(PT_EINVAL, "bad arguments to pt_local_create");
  *out = nullptr;
  int ndev = 0;
  LCK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return lfail(PT_EINVAL, "no such CUDA device");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  std::unique_ptr<pt_local> h(new pt_local());
  h->device = device;
  h->n_layers = n_layers;
  std::vector<int64_t> lptr{0}, uptr{0}, qin, qout;
  std::vector<int> bstart, blen;  // dissection blocks (global rows), when every layer has them
  bool blocked = true;
  std::vector<int> lcol, ucol, llev, ulev;
  std::vector<double2> lval, uval, ldinv, udinv;
  int64_t row0 = 0, u_row0 = 0;
  const int64_t nxe = layers[0].nxe;
  for (int l = 0; l < n_layers; ++l) {
    const pt_local_layer& A = layers[l];
    if (A.nxe != nxe || A.nze < 1 || A.n_layer < 1 || A.n_pml < 1 || A.dim != A.nze * A.nxe ||
        A.nze != A.n_layer + 2 * A.n_pml || !A.l_ptr || !A.u_ptr || !A.q_in || !A.q_out)
      return lfail(PT_EINVAL, "inconsistent local layer geometry");
    LayerDev d{};
    d.row0 = row0;
    d.dim = A.dim;
    d.nze = (int32_t)A.nze;
    d.nxe = (int32_t)A.nxe;
    d.n_layer = (int32_t)A.n_layer;
    d.n_pml = (int32_t)A.n_pml;
    d.f_row0 = A.n_pml + u_row0;  // extended-grid row of the layer's depth 1
    d.u_row0 = u_row0;
    d.has_top = l >= 1;
    d.has_bot = l <= n_layers - 2;
    d.top = 2 * (l - 1);
    d.bot = 2 * l;
    h->host_layers.push_back(d);
    int rc;
    if ((rc = split_factor(A.l_ptr, A.l_col, A.l_val, A.dim, row0, true, lptr, lcol, lval, ldinv, llev)))
      return rc;
    if ((rc = split_factor(A.u_ptr, A.u_col, A.u_val, A.dim, row0, false, uptr, ucol, uval, udinv, ulev)))
      return rc;
    if (A.n_blocks > 0 && A.block_ptr) {
      if (A.block_ptr[0] != 0 || A.block_ptr[A.n_blocks] != A.dim)
        return lfail(PT_EINVAL, "dissection blocks do not cover the layer");
      for (int64_t k = 0; k < A.n_blocks; ++k) {
        const int64_t n = A.block_ptr[k + 1] - A.block_ptr[k];
        if (n < 1 || n > TRSV_BLOCK_MAX) {
          blocked = false;  // a block the kernel cannot stage: row solve instead
          break;
        }
        bstart.push_back((int)(row0 + A.block_ptr[k]));
        blen.push_back((int)n);
      }
    } else {
      blocked = false;
    }
    for (int64_t k = 0; k < A.dim; ++k) {
      if (A.q_in[k] < 0 || A.q_in[k] >= A.dim || A.q_out[k] < 0 || A.q_out[k] >= A.dim)
        return lfail(PT_EINVAL, "local permutation out of range");
      qin.push_back(A.q_in[k]);
      qout.push_back(A.q_out[k]);
    }
    row0 += A.dim;
    u_row0 += A.n_layer;
  }
  if (row0 > INT32_MAX) return lfail(PT_EINVAL, "too many local unknowns");
  h->rows = row0;
  h->nz = u_row0;
  h->nxe = nxe;
  h->factor_nnz = (int64_t)lval.size() + (int64_t)uval.size() + 2 * row0;
  std::vector<int> lord = level_order(llev, &h->l_levels), uord = level_order(ulev, &h->u_levels);
  if (const char* e = std::getenv("PT_TRSV_BLOCK")) blocked = blocked && std::atoi(e) != 0;
  std::vector<int> lbord, ubord, lqw, uqw, llq0, ulq0, lqlev, uqlev;
  std::vector<int64_t> lboff, uboff;
  std::vector<double2> lbinv, ubinv;
  if (blocked) {
    std::vector<int> bid(row0, -1);
    for (size_t k = 0; k < bstart.size(); ++k)
      for (int i = 0; i < blen[k]; ++i) bid[bstart[k] + i] = (int)k;
    for (size_t k = 0; k < bstart.size(); ++k) {
      lboff.push_back((int64_t)lbinv.size());
      invert_block(lptr, lcol, lval, ldinv, bstart[k], blen[k], true, lbinv);
      uboff.push_back((int64_t)ubinv.size());
      invert_block(uptr, ucol, uval, udinv, bstart[k], blen[k], false, ubinv);
    }
    lbord = block_queue(lptr, lcol, bstart, blen, bid, true, &h->l_blevels, lqw);
    ubord = block_queue(uptr, ucol, bstart, blen, bid, false, &h->u_blevels, uqw);
    // warp prefix: the leading levels whose blocks all have <= 32 rows (at
    // most 32 levels); the CTA kernel's waits then count past the split
    auto warp_prefix = [&](const std::vector<int>& bord, std::vector<int>& qw, std::vector<int>& lq0,
                           std::vector<int>& qlev, int* wlev, int* split) {
      lq0.assign(1, 0);
      int q = 0;
      const int nb = (int)bord.size();
      // opt-in (PT_TRSV_WARP=1): measured slower at c3 (Newton 7.7 vs 5.5 ms),
      // the large separator blocks of the upper levels dominate
      const bool on = std::getenv("PT_TRSV_WARP") && std::atoi(std::getenv("PT_TRSV_WARP")) == 1;
      while (on && q < nb && (int)lq0.size() <= 32) {
        int e = q;
        bool small = true;
        for (; e < nb && qw[e] == qw[q]; ++e)
          if (blen[bord[e]] > TRSV_WARP_MAX) small = false;
        if (!small) break;
        q = e;
        lq0.push_back(q);
      }
      *wlev = (int)lq0.size() - 1;
      *split = q;
      qlev.assign(std::max(q, 1), 0);
      for (int l = 0; l < *wlev; ++l)
        for (int i = lq0[l]; i < lq0[l + 1]; ++i) qlev[i] = l;
      for (int i = q; i < nb; ++i) qw[i] -= q;
    };
    warp_prefix(lbord, lqw, llq0, lqlev, &h->l_wlev, &h->l_split);
    warp_prefix(ubord, uqw, ulq0, uqlev, &h->u_wlev, &h->u_split);
    h->nblocks = (int)bstart.size();
  }
  h->blocked = blocked;
  int rc;
  if ((rc = up(&h->layers, h->host_layers)) || (rc = up(&h->l_ptr, lptr)) || (rc = up(&h->u_ptr, uptr)) ||
      (rc = up(&h->l_col, lcol)) || (rc = up(&h->u_col, ucol)) || (rc = up(&h->l_val, lval)) ||
      (rc = up(&h->u_val, uval)) || (rc = up(&h->l_dinv, ldinv)) || (rc = up(&h->u_dinv, udinv)) ||
      (rc = up(&h->l_order, lord)) || (rc = up(&h->u_order, uord)) || (rc = up(&h->q_in, qin)) ||
      (rc = up(&h->q_out, qout)))
    return rc;
  if (blocked &&
      ((rc = up(&h->bstart, bstart)) || (rc = up(&h->blen, blen)) || (rc = up(&h->l_border, lbord)) ||
       (rc = up(&h->u_border, ubord)) || (rc = up(&h->l_qwait, lqw)) || (rc = up(&h->u_qwait, uqw)) ||
       (rc = up(&h->l_lq0, llq0)) || (rc = up(&h->u_lq0, ulq0)) ||
       (rc = up(&h->l_qlev, lqlev)) || (rc = up(&h->u_qlev, uqlev)) ||
       (rc = up(&h->l_boff, lboff)) || (rc = up(&h->u_boff, uboff)) ||
       (rc = up(&h->l_binv, lbinv)) || (rc = up(&h->u_binv, ubinv))))
    return rc;
  LCK(cudaMalloc(&h->y, row0 * sizeof(double2)));
  LCK(cudaMalloc(&h->w, row0 * sizeof(double2)));
  LCK(cudaMalloc(&h->z, row0 * sizeof(double2)));
  LCK(cudaMalloc(&h->flag, 2 * row0 * sizeof(int)));
  LCK(cudaMemset(h->flag, 0, 2 * row0 * sizeof(int)));
  LCK(cudaMalloc(&h->head, (4 + 64 + 2) * sizeof(int)));
  int nsm = 0, occ = 0;
  LCK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
  LCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_trsv, 1024, 0));
  int per_sm = 1;  // one block of 32 warps per SM (measured faster than two at c3)
  if (const char* e = std::getenv("PT_TRSV_BLOCKS")) per_sm = std::max(1, std::min(std::max(occ, 1), std::atoi(e)));
  if (const char* e = std::getenv("PT_TRSV_SPIN")) h->spin_ns = std::max(0, std::atoi(e));
  if (const char* e = std::getenv("PT_TRSV_CHUNK")) h->chunk = std::max(1, std::atoi(e));
  h->grid = nsm * per_sm;  // every warp resident: spinning warps never block a producer
  int bocc = 0;
  LCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bocc, k_trsv_block, TRSV_BLOCK_THREADS, 0));
  h->bgrid = nsm * std::max(bocc, 1);  // all resident: a waiting block never blocks its producers
  int wocc = 0;
  LCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&wocc, k_trsv_warp, 256, 0));
  h->wgrid = nsm * std::max(wocc, 1);
  cudaSetDevice(prev);
  *out = h.release();
  return 0;
}

int pt_local_destroy(pt_local* h) {
  if (!h) return 0;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  delete h;
  cudaSetDevice(prev);
  return 0;
}

int pt_local_info(const pt_local* h, int64_t* rows, int64_t* factor_nnz, int32_t* l_levels,
                  int32_t* u_levels) {
  if (!h) return lfail(PT_EINVAL, "null handle");
  if (rows) *rows = h->rows;
  if (factor_nnz) *factor_nnz = h->factor_nnz;
  if (l_levels) *l_levels = h->blocked ? h->l_blevels : h->l_levels;
  if (u_levels) *u_levels = h->blocked ? h->u_blevels : h->u_levels;
  return 0;
}

int pt_local_solve(pt_local* h, const double* b, double* x, pt_stream stream) {
  if (!h || !b || !x) return lfail(PT_EINVAL, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  count_launch();
  k_gather<<<elem_grid(h->rows), 256, 0, s>>>(h->q_in, h->layers, h->n_layers, h->rows,
                                              (const double2*)b, h->y);
  int rc = solve_all(h, s);
  if (!rc) {
    count_launch();
    k_gather<<<elem_grid(h->rows), 256, 0, s>>>(h->q_out, h->layers, h->n_layers, h->rows, h->z,
                                                (double2*)x);
  }
  cudaError_t e = cudaGetLastError();
  cudaSetDevice(prev);
  if (rc) return rc;
  if (e != cudaSuccess) return lfail(PT_ECUDA, cudaGetErrorString(e));
  return 0;
}

int pt_local_newton(pt_local* h, const double* f, double* traces, double* rhs, int32_t jump,
                    pt_stream stream) {
  if (!h || !f || (!traces && !rhs)) return lfail(PT_EINVAL, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  count_launch();
  k_gather_rhs<<<elem_grid(h->rows), 256, 0, s>>>(h->layers, h->n_layers, h->q_in, h->rows,
                                                  (const double2*)f, nullptr, 0, 0.0, h->y);
  int rc = solve_all(h, s);
  double2* nw = (double2*)traces;
  if (!rc && !nw) {
    if (!h->newton) {
      if (cudaMalloc(&h->newton, (size_t)h->n_layers * 4 * h->nxe * sizeof(double2)) != cudaSuccess)
        rc = lfail(PT_ECUDA, "allocation of the Newton traces failed");
    }
    nw = h->newton;
  }
  if (!rc) {
    count_launch();
    k_newton_out<<<dim3((unsigned)((h->nxe + 127) / 128), h->n_layers, 4), 128, 0, s>>>(
        h->layers, h->n_layers, h->q_out, h->z, nw);
    if (rhs) {
      const int64_t nt_m = (int64_t)(2 * h->n_layers - 2) * h->nxe;
      count_launch();
      k_polarized_rhs<<<elem_grid(2 * nt_m), 256, 0, s>>>(nw, h->n_layers, (int)h->nxe, nt_m,
                                                          jump ? 1 : 0, (double2*)rhs);
    }
  }
  cudaError_t e = cudaGetLastError();
  cudaSetDevice(prev);
  if (rc) return rc;
  if (e != cudaSuccess) return lfail(PT_ECUDA, cudaGetErrorString(e));
  return 0;
}

int pt_local_reconstruct(pt_local* h, const double* f, const double* x, double hstep, double* u,
                         pt_stream stream) {
  if (!h || !f || !x || !u || !(hstep > 0.0)) return lfail(PT_EINVAL, "bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  const int64_t nt_m = (int64_t)(2 * h->n_layers - 2) * h->nxe;
  count_launch();
  k_gather_rhs<<<elem_grid(h->rows), 256, 0, s>>>(h->layers, h->n_layers, h->q_in, h->rows,
                                                  (const double2*)f, (const double2*)x, nt_m,
                                                  1.0 / (hstep * hstep), h->y);
  int rc = solve_all(h, s);
  if (!rc) {
    count_launch();
    k_volume_out<<<dim3(64, h->n_layers), 256, 0, s>>>(h->layers, h->n_layers, h->q_out, h->z,
                                                       (double2*)u);
  }
  cudaError_t e = cudaGetLastError();
  cudaSetDevice(prev);
  if (rc) return rc;
  if (e != cudaSuccess) return lfail(PT_ECUDA, cudaGetErrorString(e));
  return 0;
}

}  // extern "C"
