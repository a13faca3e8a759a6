// Microbenchmark (profiling aid): consumer compute of one T_PLR ring piece
// (Vt rows . staged source slice) from shared memory, as the executor's
// consumers do it (no producer, no HBM).  Cycles per piece, 512 consumer
// threads, 1 CTA per SM.  Variants: lanes per row, accumulators per lane.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/piece_bench tools/piece_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
struct Item { unsigned short poff, lo, hi, n; };
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
constexpr int C = 512;
template <int LANES, int ACC>
__global__ void __launch_bounds__(C, 1) tbench(double2* out, int rows, int n, int reps, long long* cyc) {
  extern __shared__ double2 sm[];
  double2* buf = sm;
  double2* x = sm + rows * n;
  Item* items = (Item*)(x + 1024);
  for (int i = threadIdx.x; i < rows * n + 1024; i += C) sm[i] = make_double2(1e-3 * i, 1.0);
  for (int r = threadIdx.x; r < rows; r += C) items[r] = Item{(unsigned short)(r * n), 0, 0, (unsigned short)n};
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
#pragma unroll
          for (int k = 0; k < ACC; ++k) acc[k] = cfma(V[c + k * LANES], xx[c + k * LANES], acc[k]);
        }
        for (int k = 0; c < itm.n; c += LANES, ++k) acc[0] = cfma(V[c], xx[c], acc[0]);
      }
#pragma unroll
      for (int k = 1; k < ACC; ++k) { acc[0].x += acc[k].x; acc[0].y += acc[k].y; }
#pragma unroll
      for (int o = LANES >> 1; o > 0; o >>= 1) {
        acc[0].x += __shfl_xor_sync(0xffffffffu, acc[0].x, o);
        acc[0].y += __shfl_xor_sync(0xffffffffu, acc[0].y, o);
      }
      if (r < rows && sub == 0) __stcg(out + r + it, acc[0]);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(C) : "memory");
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - c0;
}
template <int L, int A>
void run(double2* out, long long* cyc, int rows, int n) {
  cudaFuncSetAttribute(tbench<L, A>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  const int reps = 1000;
  tbench<L, A><<<148, C, 200000>>>(out, rows, n, reps, cyc);
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("rows %3d n %3d lanes %2d acc %d: %6.0f cycles/piece  %.1f B/cycle (%s)\n", rows, n, L, A,
         (double)h / reps, rows * n * 16.0 / ((double)h / reps), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  double2* out; long long* cyc; cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8 * 148);
  int cfg[][2] = {{46, 55}, {23, 110}, {11, 220}, {5, 440}};
  for (auto& c : cfg) {
    run<8, 1>(out, cyc, c[0], c[1]);
    run<4, 1>(out, cyc, c[0], c[1]);
    run<4, 2>(out, cyc, c[0], c[1]);
    run<2, 2>(out, cyc, c[0], c[1]);
    run<16, 1>(out, cyc, c[0], c[1]);
    run<32, 1>(out, cyc, c[0], c[1]);
  }
}
