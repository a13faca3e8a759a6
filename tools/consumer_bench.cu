// Microbenchmark (profiling aid): consumer compute of one ring piece from
// shared memory, as the executor's 512 consumer threads do it -- T_PLR (Vt
// rows . staged source slice) and Y_PLR (a 16-row tile of U columns times t)
// -- current code against variants.  Cycles per piece (incl. the end-of-task
// barrier), 1 CTA per SM, no producer and no HBM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/consumer_bench tools/consumer_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
struct Item { unsigned short poff, lo, hi, n; };
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
constexpr int C = 512;
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"n"(C) : "memory"); }

// ---- T: current executor code (runtime lanes, one accumulator) ----------------
__global__ void __launch_bounds__(C, 1) t_cur(double2* out, int rows, int n, int lanes, int reps, long long* cyc) {
  extern __shared__ double2 sm[];
  double2* buf = sm;
  double2* x = sm + rows * n;
  Item* items = (Item*)(x + 1024);
  for (int i = threadIdx.x; i < rows * n + 1024; i += C) sm[i] = make_double2(1e-3 * i, 1.0);
  for (int r = threadIdx.x; r < rows; r += C) items[r] = Item{(unsigned short)(r * n), (unsigned short)(r % 3), 0, (unsigned short)n};
  __syncthreads();
  long long c0 = clock64();
  const int lsh = __ffs(lanes) - 1;
  const int sub = threadIdx.x & (lanes - 1);
  for (int it = 0; it < reps; ++it) {
    for (int base = 0; base < rows; base += C >> lsh) {
      const int r = base + (int)(threadIdx.x >> lsh);
      double2 acc = make_double2(0.0, 0.0);
      if (r < rows) {
        const Item itm = items[r];
        const double2* V = buf + itm.poff;
        const double2* xx = x + itm.lo;
        for (int c = sub; c < itm.n; c += lanes) acc = cfma(V[c], xx[c], acc);
      }
      for (int o = lanes >> 1; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if (r < rows && sub == 0) __stcg(out + r + it, acc);
    }
    csync();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - c0;
}

// ---- T variant: compile-time lanes, ACC independent accumulators ------------------
template <int LANES, int ACC>
__global__ void __launch_bounds__(C, 1) t_var(double2* out, int rows, int n, int reps, long long* cyc) {
  extern __shared__ double2 sm[];
  double2* buf = sm;
  double2* x = sm + rows * n;
  Item* items = (Item*)(x + 1024);
  for (int i = threadIdx.x; i < rows * n + 1024; i += C) sm[i] = make_double2(1e-3 * i, 1.0);
  for (int r = threadIdx.x; r < rows; r += C) items[r] = Item{(unsigned short)(r * n), (unsigned short)(r % 3), 0, (unsigned short)n};
  __syncthreads();
  long long c0 = clock64();
  const int sub = threadIdx.x & (LANES - 1);
  for (int it = 0; it < reps; ++it) {
    for (int base = 0; base < rows; base += C / LANES) {
      const int r = base + (int)threadIdx.x / LANES;
      double2 acc[ACC];
#pragma unroll
      for (int k = 0; k < ACC; ++k) acc[k] = make_double2(0.0, 0.0);
      if (r < rows) {
        const Item itm = items[r];
        const double2* V = buf + itm.poff;
        const double2* xx = x + itm.lo;
        int c = sub;
        for (; c + (ACC - 1) * LANES < itm.n; c += ACC * LANES) {
          double2 v[ACC], w[ACC];
#pragma unroll
          for (int k = 0; k < ACC; ++k) { v[k] = V[c + k * LANES]; w[k] = xx[c + k * LANES]; }
#pragma unroll
          for (int k = 0; k < ACC; ++k) acc[k] = cfma(v[k], w[k], acc[k]);
        }
#pragma unroll
        for (int k = 0; k < ACC - 1; ++k)
          if (c + k * LANES < itm.n) acc[k] = cfma(V[c + k * LANES], xx[c + k * LANES], acc[k]);
      }
#pragma unroll
      for (int k = 1; k < ACC; ++k) acc[0] = cadd(acc[0], acc[k]);
#pragma unroll
      for (int o = LANES >> 1; o > 0; o >>= 1) {
        acc[0].x += __shfl_xor_sync(0xffffffffu, acc[0].x, o);
        acc[0].y += __shfl_xor_sync(0xffffffffu, acc[0].y, o);
      }
      if (r < rows && sub == 0) __stcg(out + r + it, acc[0]);
    }
    csync();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - c0;
}

// ---- Y: current executor code ------------------------------------------------
// ncol flat columns of up to 16 rows each (tile-major U); thread (r, g), 32
// groups; two columns per iteration into two accumulators; partials through
// smem, 16 threads add the 32 group sums in order.
__global__ void __launch_bounds__(C, 1) y_cur(double2* out, int ncol, int reps, long long* cyc) {
  extern __shared__ double2 sm[];
  constexpr int G = C / 16;
  double2* buf = sm;                 // ncol * 16
  double2* vec = sm + ncol * 16;     // ncol
  double2* part = vec + 1024;        // 512
  Item* items = (Item*)(part + 512);
  for (int i = threadIdx.x; i < ncol * 16 + 1024; i += C) sm[i] = make_double2(1e-3 * i, 1.0);
  for (int f = threadIdx.x; f < ncol; f += C) items[f] = Item{(unsigned short)(f * 16), 0, 16, 0};
  __syncthreads();
  long long c0 = clock64();
  const int r = threadIdx.x % 16, g = threadIdx.x / 16;
  for (int it = 0; it < reps; ++it) {
    double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
    int f = g;
    for (; f + G < ncol; f += 2 * G) {
      Item i0 = items[f], i1 = items[f + G];
      double2 t0 = vec[f], t1 = vec[f + G];
      double2 u0 = (r >= i0.lo && r < i0.hi) ? buf[i0.poff + (r - i0.lo)] : make_double2(0.0, 0.0);
      double2 u1 = (r >= i1.lo && r < i1.hi) ? buf[i1.poff + (r - i1.lo)] : make_double2(0.0, 0.0);
      acc = cfma(u0, t0, acc);
      acc2 = cfma(u1, t1, acc2);
    }
    for (; f < ncol; f += G) {
      Item i0 = items[f];
      if (r >= i0.lo && r < i0.hi) acc = cfma(buf[i0.poff + (r - i0.lo)], vec[f], acc);
    }
    part[g * 16 + r] = cadd(acc, acc2);
    csync();
    if (threadIdx.x < 16) {
      double2 v = make_double2(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < G; ++i) v = cadd(v, part[i * 16 + threadIdx.x]);
      __stcg(out + threadIdx.x + it, v);
    }
    csync();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - c0;
}

// ---- Y variant: U columns unrolled by UN, shuffle pre-reduction of the two
// groups of a warp, 16 warp partials added by 16 threads ------------------------
template <int UN>
__global__ void __launch_bounds__(C, 1) y_var(double2* out, int ncol, int reps, long long* cyc) {
  extern __shared__ double2 sm[];
  constexpr int G = C / 16;
  double2* buf = sm;
  double2* vec = sm + ncol * 16;
  double2* part = vec + 1024;
  Item* items = (Item*)(part + 512);
  for (int i = threadIdx.x; i < ncol * 16 + 1024; i += C) sm[i] = make_double2(1e-3 * i, 1.0);
  for (int f = threadIdx.x; f < ncol; f += C) items[f] = Item{(unsigned short)(f * 16), 0, 16, 0};
  __syncthreads();
  long long c0 = clock64();
  const int r = threadIdx.x % 16, g = threadIdx.x / 16;
  for (int it = 0; it < reps; ++it) {
    double2 acc[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    int f = g;
    for (; f + (UN - 1) * G < ncol; f += UN * G) {
      Item im[UN];
      double2 t[UN], u[UN];
#pragma unroll
      for (int k = 0; k < UN; ++k) { im[k] = items[f + k * G]; t[k] = vec[f + k * G]; }
#pragma unroll
      for (int k = 0; k < UN; ++k)
        u[k] = (r >= im[k].lo && r < im[k].hi) ? buf[im[k].poff + (r - im[k].lo)] : make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < UN; ++k) acc[k & 1] = cfma(u[k], t[k], acc[k & 1]);
    }
    for (; f < ncol; f += G) {
      Item i0 = items[f];
      if (r >= i0.lo && r < i0.hi) acc[0] = cfma(buf[i0.poff + (r - i0.lo)], vec[f], acc[0]);
    }
    double2 v = cadd(acc[0], acc[1]);
    v.x += __shfl_xor_sync(0xffffffffu, v.x, 16);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, 16);
    if ((threadIdx.x & 31) < 16) part[(threadIdx.x >> 5) * 16 + r] = v;
    csync();
    if (threadIdx.x < 16) {
      double2 s[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
#pragma unroll
      for (int i = 0; i < 16; ++i) s[i & 3] = cadd(s[i & 3], part[i * 16 + threadIdx.x]);
      __stcg(out + threadIdx.x + it, cadd(cadd(s[0], s[1]), cadd(s[2], s[3])));
    }
    csync();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - c0;
}


// ---- T variant: R consecutive rows of one leaf per lane group (x loaded once per
// column for R rows), LANES lanes per row group --------------------------------------
template <int LANES, int R>
__global__ void __launch_bounds__(C, 1) t_rows(double2* out, int rows, int n, int reps, long long* cyc) {
  extern __shared__ double2 sm[];
  double2* buf = sm;
  double2* x = sm + rows * n;
  for (int i = threadIdx.x; i < rows * n + 1024; i += C) sm[i] = make_double2(1e-3 * i, 1.0);
  __syncthreads();
  long long c0 = clock64();
  const int sub = threadIdx.x & (LANES - 1);
  const int groups = (rows + R - 1) / R;
  for (int it = 0; it < reps; ++it) {
    for (int base = 0; base < groups; base += C / LANES) {
      const int gi = base + (int)threadIdx.x / LANES;
      double2 acc[R];
#pragma unroll
      for (int k = 0; k < R; ++k) acc[k] = make_double2(0.0, 0.0);
      const int r0 = gi * R;
      if (gi < groups) {
        const double2* V = buf + r0 * n;
        const double2* xx = x + (r0 % 3);
        const int nr = min(R, rows - r0);
        for (int c = sub; c < n; c += LANES) {
          const double2 xv = xx[c];
#pragma unroll
          for (int k = 0; k < R; ++k)
            if (k < nr) acc[k] = cfma(V[k * n + c], xv, acc[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < R; ++k)
#pragma unroll
        for (int o = LANES >> 1; o > 0; o >>= 1) {
          acc[k].x += __shfl_xor_sync(0xffffffffu, acc[k].x, o);
          acc[k].y += __shfl_xor_sync(0xffffffffu, acc[k].y, o);
        }
      if (gi < groups && sub == 0)
#pragma unroll
        for (int k = 0; k < R; ++k)
          if (r0 + k < rows) __stcg(out + r0 + k + it, acc[k]);
    }
    csync();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - c0;
}

// ---- Y variant: RP rows per thread (rows r, r + 16/RP, ...), 16/RP row slots x
// (32*RP) column groups; items and t loaded once per column for RP rows ----------
template <int RP>
__global__ void __launch_bounds__(C, 1) y_rows(double2* out, int ncol, int reps, long long* cyc) {
  extern __shared__ double2 sm[];
  constexpr int RS = 16 / RP, G = C / RS;
  double2* buf = sm;
  double2* vec = sm + ncol * 16;
  double2* part = vec + 1024;
  Item* items = (Item*)(part + 2048);
  for (int i = threadIdx.x; i < ncol * 16 + 1024; i += C) sm[i] = make_double2(1e-3 * i, 1.0);
  for (int f = threadIdx.x; f < ncol; f += C) items[f] = Item{(unsigned short)(f * 16), 0, 16, 0};
  __syncthreads();
  long long c0 = clock64();
  const int r = threadIdx.x % RS, g = threadIdx.x / RS;
  for (int it = 0; it < reps; ++it) {
    double2 acc[RP];
#pragma unroll
    for (int k = 0; k < RP; ++k) acc[k] = make_double2(0.0, 0.0);
    for (int f = g; f < ncol; f += G) {
      const Item im = items[f];
      const double2 t = vec[f];
#pragma unroll
      for (int k = 0; k < RP; ++k) {
        const int rr = r + k * RS;
        if (rr >= im.lo && rr < im.hi) acc[k] = cfma(buf[im.poff + (rr - im.lo)], t, acc[k]);
      }
    }
    // reduce over the G column groups: warp = 32/RS groups
#pragma unroll
    for (int k = 0; k < RP; ++k)
      for (int o = RS; o < 32; o <<= 1) {
        acc[k].x += __shfl_xor_sync(0xffffffffu, acc[k].x, o);
        acc[k].y += __shfl_xor_sync(0xffffffffu, acc[k].y, o);
      }
    if ((threadIdx.x & 31) < RS)
#pragma unroll
      for (int k = 0; k < RP; ++k) part[(threadIdx.x >> 5) * 16 + r + k * RS] = acc[k];
    csync();
    if (threadIdx.x < 16) {
      double2 s4[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
#pragma unroll
      for (int i = 0; i < 16; ++i) s4[i & 3] = cadd(s4[i & 3], part[i * 16 + threadIdx.x]);
      __stcg(out + threadIdx.x + it, cadd(cadd(s4[0], s4[1]), cadd(s4[2], s4[3])));
    }
    csync();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - c0;
}


// T variant with NT threads (occupancy test)
template <int LANES, int NT>
__global__ void __launch_bounds__(NT, 1) t_occ(double2* out, int rows, int n, int reps, long long* cyc) {
  extern __shared__ double2 sm[];
  double2* buf = sm;
  double2* x = sm + rows * n;
  Item* items = (Item*)(x + 1024);
  for (int i = threadIdx.x; i < rows * n + 1024; i += NT) sm[i] = make_double2(1e-3 * i, 1.0);
  for (int r = threadIdx.x; r < rows; r += NT) items[r] = Item{(unsigned short)(r * n), (unsigned short)(r % 3), 0, (unsigned short)n};
  __syncthreads();
  long long c0 = clock64();
  const int sub = threadIdx.x & (LANES - 1);
  for (int it = 0; it < reps; ++it) {
    for (int base = 0; base < rows; base += NT / LANES) {
      const int r = base + (int)threadIdx.x / LANES;
      double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
      if (r < rows) {
        const Item itm = items[r];
        const double2* V = buf + itm.poff;
        const double2* xx = x + itm.lo;
        int c = sub;
        for (; c + LANES < itm.n; c += 2 * LANES) {
          acc = cfma(V[c], xx[c], acc);
          acc2 = cfma(V[c + LANES], xx[c + LANES], acc2);
        }
        if (c < itm.n) acc = cfma(V[c], xx[c], acc);
      }
      acc = cadd(acc, acc2);
#pragma unroll
      for (int o = LANES >> 1; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if (r < rows && sub == 0) __stcg(out + r + it, acc);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - c0;
}
// empty variant: only the loads (sum of V), no x, no FMA chain
template <int LANES>
__global__ void __launch_bounds__(512, 1) t_loads(double2* out, int rows, int n, int reps, long long* cyc) {
  extern __shared__ double2 sm[];
  double2* buf = sm;
  for (int i = threadIdx.x; i < rows * n + 1024; i += 512) sm[i] = make_double2(1e-3 * i, 1.0);
  __syncthreads();
  long long c0 = clock64();
  const int sub = threadIdx.x & (LANES - 1);
  double s = 0;
  for (int it = 0; it < reps; ++it) {
    for (int base = 0; base < rows; base += 512 / LANES) {
      const int r = base + (int)threadIdx.x / LANES;
      if (r < rows) {
        const double2* V = buf + r * n;
        for (int c = sub; c < n; c += LANES) s += V[c].x;
      }
    }
    __syncthreads();
  }
  if (s == 1.2345) out[0].x = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - c0;
}

long long* g_cyc;
double2* g_out;
const int REPS = 2000;
template <typename K, typename... A>
double run_nt(K kern, int nt, size_t smem, A... a) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  kern<<<148, nt, smem>>>(g_out, a..., REPS, g_cyc);
  long long h;
  cudaMemcpy(&h, g_cyc, 8, cudaMemcpyDeviceToHost);
  if (cudaGetLastError() != cudaSuccess) printf("error\n");
  return (double)h / REPS;
}
template <typename K, typename... A>
double run(K kern, size_t smem, A... a) { return run_nt(kern, C, smem, a...); }
int main() {
  cudaMalloc(&g_out, 1 << 24);
  cudaMalloc(&g_cyc, 8 * 148);
  int tcfg[][3] = {{52, 55, 8}, {26, 110, 16}, {13, 220, 32}, {6, 440, 32}};
  for (auto& c : tcfg) {
    const int rows = c[0], n = c[1], ln = c[2];
    const double B = rows * n * 16.0;
    printf("T piece %2d x %3d (%5.1f KB): current(lanes %2d) %5.0f cyc", rows, n, B / 1024, ln,
           run(t_cur, 200000, rows, n, ln));
    printf(" | rows L8R2 %5.0f L8R4 %5.0f L16R2 %5.0f L16R4 %5.0f L32R2 %5.0f L32R4 %5.0f L4R4 %5.0f\n",
           run(t_rows<8, 2>, 200000, rows, n), run(t_rows<8, 4>, 200000, rows, n),
           run(t_rows<16, 2>, 200000, rows, n), run(t_rows<16, 4>, 200000, rows, n),
           run(t_rows<32, 2>, 200000, rows, n), run(t_rows<32, 4>, 200000, rows, n),
           run(t_rows<4, 4>, 200000, rows, n));
  }
  for (auto& c : tcfg) {
    const int rows = c[0], n = c[1];
    printf("T %2d x %3d occupancy: L8 256thr %5.0f 512thr %5.0f 1024thr %5.0f | L16 512 %5.0f 1024 %5.0f | loads-only L8 %5.0f L16 %5.0f\n", rows, n,
           run_nt(t_occ<8, 256>, 256, 200000, rows, n), run_nt(t_occ<8, 512>, 512, 200000, rows, n),
           run_nt(t_occ<8, 1024>, 1024, 200000, rows, n), run_nt(t_occ<16, 512>, 512, 200000, rows, n),
           run_nt(t_occ<16, 1024>, 1024, 200000, rows, n), run(t_loads<8>, 200000, rows, n), run(t_loads<16>, 200000, rows, n));
  }
  for (int ncol : {64, 128, 180, 256}) {
    printf("Y tile 16 x %3d cols (%5.1f KB): current %5.0f cyc | UN2 %5.0f | RP2 %5.0f RP4 %5.0f RP8 %5.0f\n", ncol,
           ncol * 256.0 / 1024, run(y_cur, 200000, ncol), run(y_var<2>, 200000, ncol),
           run(y_rows<2>, 200000, ncol), run(y_rows<4>, 200000, ncol), run(y_rows<8>, 200000, ncol));
  }
  return 0;
}
