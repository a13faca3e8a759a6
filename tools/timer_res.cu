// Resolution of %globaltimer vs clock64 on this GPU (profiling aid).
#include <cstdio>
__global__ void k(unsigned long long* out) {
  unsigned long long prev, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
  int n = 0;
  long long c0 = clock64();
  while (n < 16) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != prev) { out[n++] = t - prev; prev = t; }
  }
  out[16] = clock64() - c0;
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 17 * 8);
  k<<<1, 1>>>(d);
  unsigned long long h[17]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("globaltimer steps (ns):"); for (int i = 0; i < 16; ++i) printf(" %llu", h[i]);
  printf("\ncycles for 16 steps: %llu\n", h[16]);
}
