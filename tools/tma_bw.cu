// Microbenchmark (profiling aid): HBM -> smem streaming with TMA bulk copies.
// Each CTA streams `chunks` contiguous chunks of `bytes` with `depth` copies
// in flight (ring of `depth` smem buffers, one mbarrier each) and touches the
// data (sum) so the copies are consumed.  Reports GB/s for grid = SMs * ctas.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bw tools/tma_bw.cu
//   ./tma_bw <ctas_per_sm> <chunk_bytes> <depth> [total_MB]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void stream(const double2* __restrict__ src, size_t chunk_elems, int chunks_per_cta,
                       int depth, double* out, int off, int scatter) {
  extern __shared__ __align__(128) double2 buf[];
  __shared__ __align__(8) unsigned long long bar[8];
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t base = (size_t)blockIdx.x * chunks_per_cta * (chunk_elems + off) + off;
  const unsigned bytes = (unsigned)(chunk_elems * sizeof(double2));
  auto issue = [&](int c) {
    const int s = c % depth;
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                     "r"(su32(buf + s * chunk_elems)), "l"(src + (scatter ? (((size_t)(c * 7919 + blockIdx.x * 104729) % ((size_t)gridDim.x * chunks_per_cta)) * (chunk_elems + off) + off) : base + (size_t)c * (chunk_elems + off))), "r"(bytes),
                 "r"(su32(&bar[s])));
  };
  if (threadIdx.x == 0)
    for (int c = 0; c < depth && c < chunks_per_cta; ++c) issue(c);
  double acc = 0.0;
  unsigned phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int c = 0; c < chunks_per_cta; ++c) {
    const int s = c % depth;
    unsigned done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}"
                   : "=r"(done) : "r"(su32(&bar[s])), "r"(phase[s]));
    phase[s] ^= 1u;
    const double2* b = buf + s * chunk_elems;
    for (size_t i = threadIdx.x; i < chunk_elems; i += blockDim.x) acc += b[i].x;
    __syncthreads();
    if (threadIdx.x == 0 && c + depth < chunks_per_cta) issue(c + depth);
  }
  if (acc == 12345.678) out[0] = acc;
}

int main(int argc, char** argv) {
  const int cps = argc > 1 ? atoi(argv[1]) : 3;
  const size_t bytes = argc > 2 ? atol(argv[2]) : 23 * 1024;
  const int depth = argc > 3 ? atoi(argv[3]) : 2;
  const size_t total_mb = argc > 4 ? atol(argv[4]) : 600;
  const int off = argc > 5 ? atoi(argv[5]) : 0;
  const int scatter = argc > 6 ? atoi(argv[6]) : 0;
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = nsm * cps;
  const size_t chunk_elems = bytes / 16;
  const int chunks = (int)((total_mb << 20) / (bytes * grid));
  const size_t n = (size_t)grid * chunks * (chunk_elems + off) + 64;
  double2* src;
  double* out;
  cudaMalloc(&src, n * 16);
  cudaMalloc(&out, 8);
  cudaMemset(src, 0, n * 16);
  const size_t smem = depth * bytes;
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stream, 256, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) stream<<<grid, 256, smem>>>(src, chunk_elems, chunks, depth, out, off, scatter);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int it = 0; it < reps; ++it) stream<<<grid, 256, smem>>>(src, chunk_elems, chunks, depth, out, off, scatter);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double gbs = (double)grid * chunks * bytes * reps / (ms * 1e-3) / 1e9;
  printf("ctas/sm %d (occ %d) chunk %zu B depth %d off %d scatter %d: %.0f GB/s  (%s)\n", cps, occ, bytes, depth, off, scatter, gbs,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
