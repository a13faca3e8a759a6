// Microbenchmark (profiling aid): FP64 tensor-core (DMMA, mma.sync .f64)
// throughput per SM vs plain DFMA on this GPU, to size the multi-RHS
// (batched) contraction tiles.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma884(double* d, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma16816(double* d, const double* a, const double* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
      "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

__global__ void k884(double* out, int n, long long* cyc) {
  double acc[8][2] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  __syncthreads();
  long long c0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int u = 0; u < 8; ++u) mma884(acc[u], a, b);
  __syncthreads();
  long long c1 = clock64();
  double s = 0;
  for (int u = 0; u < 8; ++u) s += acc[u][0] + acc[u][1];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}
__global__ void k16816(double* out, int n, long long* cyc) {
  double acc[4][4] = {};
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-6;
  __syncthreads();
  long long c0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int u = 0; u < 4; ++u) mma16816(acc[u], a, b);
  __syncthreads();
  long long c1 = clock64();
  double s = 0;
  for (int u = 0; u < 4; ++u) s += acc[u][0] + acc[u][1] + acc[u][2] + acc[u][3];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}
__global__ void kfma(double* out, int n, long long* cyc) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  const double b = 1.0000001, c = 1e-9;
  __syncthreads();
  long long c0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = fma(a[u], b, c);
  __syncthreads();
  long long c1 = clock64();
  double s = 0;
  for (int u = 0; u < 8; ++u) s += a[u];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 4096 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int n = 4096;
  for (int threads : {128, 256, 512}) {
    for (int which = 0; which < 3; ++which) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (which == 0) k884<<<sms, threads>>>(out, n, cyc);
        if (which == 1) k16816<<<sms, threads>>>(out, n, cyc);
        if (which == 2) kfma<<<sms, threads>>>(out, n, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double warps = threads / 32.0;
      double flop;  // per SM
      if (which == 0) flop = warps * n * 8 * 512.0;
      else if (which == 1) flop = warps * n * 4 * 4096.0;
      else flop = threads * (double)n * 8 * 2.0;
      const char* nm[3] = {"dmma m8n8k4", "dmma m16n8k16", "dfma"};
      printf("%-14s threads %3d: %.1f flop/cycle/SM, %.2f TFLOP/s (events)\n", nm[which], threads,
             flop / c, flop * sms / (ms * 1e-3) / 1e12);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
