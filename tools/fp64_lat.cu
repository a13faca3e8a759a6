// Microbenchmark (profiling aid): FP64 FMA dependent-chain latency and
// throughput per SM on this GPU.
#include <cstdio>
__global__ void lat(double* out, int n, long long* cyc) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 1e-9;
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
  long long c1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = a;
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}
__global__ void thr(double* out, int n, long long* cyc) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 1.0000001, c = 1e-9;
  __syncthreads();
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  __syncthreads();
  long long c1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}
__global__ void shfl_lat(double* out, int n, long long* cyc) {
  double a = threadIdx.x;
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) a += __shfl_xor_sync(0xffffffffu, a, 1);
  long long c1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
}
__global__ void lds_lat(double* out, int n, long long* cyc) {
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
  __syncthreads();
  int j = threadIdx.x;
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) j = idx[j];
  long long c1 = clock64();
  out[threadIdx.x] = j;
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 22); cudaMalloc(&cyc, 8 * 1024);
  long long h; const int n = 4096;
  lat<<<1, 32>>>(out, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.1f cycles\n", (double)h / (4.0 * n));
  for (int t : {128, 256, 512, 1024}) {
    thr<<<148, t>>>(out, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA throughput, %4d threads/SM: %.1f DFMA/clk/SM\n", t, 8.0 * n * t / (double)h);
  }
  shfl_lat<<<1, 32>>>(out, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("SHFL+DADD dependent latency: %.1f cycles\n", (double)h / n);
  lds_lat<<<1, 32>>>(out, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("LDS dependent latency: %.1f cycles\n", (double)h / n);
}
