// Microbenchmark (profiling aid): does a release fence (red.release.gpu ->
// MEMBAR.ALL.GPU) issued by a warp wait for that warp's in-flight TMA bulk
// loads?  One CTA per SM: lane 0 optionally issues a 48 KB cp.async.bulk
// global->shared, then times a red.release.gpu (and, separately, a relaxed
// red) with clock64.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// with_tma: 0 none, 1 issued by the releasing warp, 2 issued by another warp
__global__ void k(const char* src, int* ctr, long long* out, int with_tma, int release) {
  extern __shared__ __align__(128) char buf[];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t bytes = 48 * 1024;
  if (with_tma == 2 && threadIdx.x == 32) {  // another warp keeps a bulk copy in flight
    for (int it = 0; it < 8; ++it) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(buf)),
                   "l"(src + ((size_t)blockIdx.x * 8 + it) * bytes), "r"(bytes), "r"(sa(&bar)) : "memory");
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(sa(&bar)), "r"(it & 1) : "memory");
    }
    return;
  }
  if (threadIdx.x != 0) return;
  if (with_tma == 2) __nanosleep(200);
  long long dt = 0;
  for (int it = 0; it < 8; ++it) {
    if (with_tma == 1) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(buf)),
                   "l"(src + ((size_t)blockIdx.x * 8 + it) * bytes), "r"(bytes), "r"(sa(&bar)) : "memory");
    }
    const long long t0 = clock64();
    if (release)
      asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(ctr + blockIdx.x) : "memory");
    else
      asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(ctr + blockIdx.x) : "memory");
    const long long t1 = clock64();
    dt += t1 - t0;
    if (with_tma == 2) __nanosleep(300);
    if (with_tma == 1) {
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(sa(&bar)), "r"(it & 1) : "memory");
    }
  }
  out[blockIdx.x] = dt / 8;
}
int main() {
  char* src; int* ctr; long long* out;
  const size_t n = (size_t)148 * 8 * 48 * 1024;
  cudaMalloc(&src, n); cudaMalloc(&ctr, 148 * 4); cudaMalloc(&out, 148 * 8);
  cudaMemset(src, 1, n); cudaMemset(ctr, 0, 148 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  long long h[148];
  for (int rep = 0; rep < 2; ++rep)
    for (int tma = 0; tma < 3; ++tma)
      for (int rel = 0; rel < 2; ++rel) {
        k<<<148, 64, 64 * 1024>>>(src, ctr, out, tma, rel);
        cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
        double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
        if (rep) printf("tma %d release %d: red issue %.0f cycles (mean over CTAs)\n", tma, rel, s / 148);
      }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
