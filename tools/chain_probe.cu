// Microbenchmarks for the sweep-chain design (profiling aid, not product code).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/chain_probe tools/chain_probe.cu
//   ./tools/chain_probe
//
// 1. max active clusters of 8 / 16 CTAs at ~200 KB smem, 640 threads;
// 2. HBM read bandwidth (TMA bulk ring) vs number of streaming CTAs;
// 3. bandwidth split when k CTAs stream with a deeper ring than the rest;
// 4. a chain of dependent hops through global memory (flag + TMA reload),
//    alone and beside CTAs that saturate HBM;
// 5. all-gather rounds inside a 16-CTA cluster (DSMEM bulk copies).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mb_init(unsigned long long* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mb_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned ph) {
  unsigned done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}"
                 : "=r"(done) : "r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(b)) : "memory");
}

// ---- 2/3: streaming ---------------------------------------------------------
// CTA b streams `per_cta` bytes of its own region with a ring of `depth`
// chunks of `chunk` bytes (depth_hi for CTAs < k_hi); records start/end.
__global__ void k_stream(const char* src, size_t per_cta, unsigned chunk, int depth, int depth_hi, int k_hi,
                         unsigned long long* t, double* sink) {
  extern __shared__ __align__(128) char buf[];
  __shared__ __align__(8) unsigned long long bar[16];
  const int d = (int)blockIdx.x < k_hi ? depth_hi : depth;
  if (threadIdx.x == 0) {
    for (int i = 0; i < d; ++i) mb_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const char* base = src + (size_t)blockIdx.x * per_cta;
  const int n = (int)(per_cta / chunk);
  if (threadIdx.x == 0) t[2 * blockIdx.x] = gtime();
  if (threadIdx.x == 0)
    for (int c = 0; c < d && c < n; ++c) {
      mb_expect(&bar[c], chunk);
      tma_load(buf + (size_t)c * chunk, base + (size_t)c * chunk, chunk, &bar[c]);
    }
  double acc = 0.0;
  for (int c = 0; c < n; ++c) {
    const int s = c % d;
    mb_wait(&bar[s], (c / d) & 1);
    const double* p = (const double*)(buf + (size_t)s * chunk);
    for (unsigned i = threadIdx.x; i < chunk / 8; i += blockDim.x) acc += p[i];
    __syncthreads();
    if (threadIdx.x == 0 && c + d < n) {
      asm volatile("fence.proxy.async.shared::cta;");
      mb_expect(&bar[s], chunk);
      tma_load(buf + (size_t)s * chunk, base + (size_t)(c + d) * chunk, chunk, &bar[s]);
    }
  }
  if (threadIdx.x == 0) t[2 * blockIdx.x + 1] = gtime();
  if (acc == 12345.678) sink[0] = acc;
}

// ---- 4: chain of hops through global memory -------------------------------------
// CTAs [0, nchain) run hops h = 0..H-1, hop h on CTA h % nchain: wait for
// flag[h - 1], TMA-load `bytes` of the previous hop's output, add, store the
// output (st.cg), fence + release flag[h].  CTAs >= nchain stream HBM.
__global__ void k_chain(double* vec, int* flags, int H, int nchain, unsigned bytes, const char* src,
                        size_t per_cta, unsigned chunk, unsigned long long* t, double* sink) {
  extern __shared__ __align__(128) char buf[];
  __shared__ __align__(8) unsigned long long bar[8];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mb_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if ((int)blockIdx.x >= nchain) {  // background streaming, depth 4
    const int d = 4;
    const char* base = src + (size_t)(blockIdx.x - nchain) * per_cta;
    const int n1 = (int)(per_cta / chunk), n = n1 * 16;  // 16 passes over the region
    if (threadIdx.x == 0)
      for (int c = 0; c < d && c < n; ++c) {
        mb_expect(&bar[c], chunk);
        tma_load(buf + (size_t)c * chunk, base + (size_t)(c % n1) * chunk, chunk, &bar[c]);
      }
    double acc = 0.0;
    for (int c = 0; c < n; ++c) {
      const int s = c % d;
      mb_wait(&bar[s], (c / d) & 1);
      const double* p = (const double*)(buf + (size_t)s * chunk);
      for (unsigned i = threadIdx.x; i < chunk / 8; i += blockDim.x) acc += p[i];
      __syncthreads();
      if (threadIdx.x == 0 && c + d < n) {
        asm volatile("fence.proxy.async.shared::cta;");
        mb_expect(&bar[s], chunk);
        tma_load(buf + (size_t)s * chunk, base + (size_t)((c + d) % n1) * chunk, chunk, &bar[s]);
      }
    }
    if (acc == 12345.678) sink[0] = acc;
    return;
  }
  const int nel = bytes / 8;
  double* stage = (double*)buf;
  int phase = 0;
  __shared__ unsigned long long t0;
  if (threadIdx.x == 0) t0 = gtime();
  for (int h = blockIdx.x; h < H; h += nchain) {
    if (h > 0) {
      if (threadIdx.x == 0) {
        int v;
        do {
          asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(flags + h - 1) : "memory");
        } while (v == 0);
        asm volatile("fence.proxy.async.global;" ::: "memory");
        mb_expect(&bar[0], bytes);
        tma_load(stage, vec + (size_t)((h - 1) & 1) * nel, bytes, &bar[0]);
      }
      mb_wait(&bar[0], phase);
      phase ^= 1;
    }
    double* out = vec + (size_t)(h & 1) * nel;
    for (int i = threadIdx.x; i < nel; i += blockDim.x) {
      const double v = (h > 0 ? stage[i] : 0.0) + 1.0;
      asm volatile("st.global.cg.f64 [%0], %1;" ::"l"(out + i), "d"(v) : "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(flags + h) : "memory");
  }
  if (threadIdx.x == 0 && blockIdx.x == (unsigned)((H - 1) % nchain)) {
    t[0] = t0;
    t[1] = gtime();
  }
}

// ---- 5: all-gather rounds in a cluster -------------------------------------------
// Every CTA of a 16-CTA cluster sends its `slice` bytes to every CTA's buffer
// (cp.async.bulk smem -> remote smem, completing on the receiver's mbarrier);
// a round ends when a CTA has received all 16 slices.
__global__ void __cluster_dims__(16, 1, 1) k_allgather(int rounds, unsigned slice, unsigned long long* t) {
  extern __shared__ __align__(128) char buf[];  // [2][16 * slice] receive, [slice] send
  __shared__ __align__(8) unsigned long long bar[2];
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    mb_init(&bar[0], 1);
    mb_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  char* send = buf + 2 * 16 * slice;
  unsigned long long t0 = gtime();
  for (int r = 0; r < rounds; ++r) {
    const int b = r & 1;
    if (threadIdx.x == 0) mb_expect(&bar[b], 16 * slice);
    // the receivers must have armed round r's barrier (and consumed round
    // r - 2's buffer) before slices land: one cluster barrier per round
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    for (unsigned i = threadIdx.x; i < slice / 8; i += blockDim.x) ((double*)send)[i] = r + rank;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 16) {
      const unsigned dst_local = su32(buf + (size_t)b * 16 * slice + rank * slice);
      const unsigned bar_local = su32(&bar[b]);
      unsigned dst, rb;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(dst_local), "r"(threadIdx.x));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(bar_local), "r"(threadIdx.x));
      asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                   "r"(su32(send)), "r"(slice), "r"(rb) : "memory");
    }
    mb_wait(&bar[b], (r >> 1) & 1);
    asm volatile("cp.async.bulk.commit_group; cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  if (threadIdx.x == 0 && rank == 0 && blockIdx.x < 16) {
    t[0] = t0;
    t[1] = gtime();
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ---- 5b: the same round without the barrier: receivers arm round r + 1 early
__global__ void __cluster_dims__(16, 1, 1) k_allgather_nb(int rounds, unsigned slice, unsigned long long* t) {
  extern __shared__ __align__(128) char buf[];
  __shared__ __align__(8) unsigned long long bar[4];
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mb_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
    mb_expect(&bar[0], 16 * slice);
    mb_expect(&bar[1], 16 * slice);
    mb_expect(&bar[2], 16 * slice);
    mb_expect(&bar[3], 16 * slice);
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  char* send = buf + 4 * 16 * slice;
  unsigned long long t0 = gtime();
  for (int r = 0; r < rounds; ++r) {
    const int b = r & 3;
    for (unsigned i = threadIdx.x; i < slice / 8; i += blockDim.x) ((double*)(send + (r & 1) * slice))[i] = r + rank;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 16) {
      const unsigned dst_local = su32(buf + (size_t)b * 16 * slice + rank * slice);
      const unsigned bar_local = su32(&bar[b]);
      unsigned dst, rb;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(dst_local), "r"(threadIdx.x));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(bar_local), "r"(threadIdx.x));
      asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                   "r"(su32(send + (r & 1) * slice)), "r"(slice), "r"(rb) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    mb_wait(&bar[b], (r >> 2) & 1);
    // re-arm this buffer for round r + 4 (all 16 slices of round r landed;
    // a sender is at most 2 rounds ahead since it waits for its own round)
    if (threadIdx.x == 0) mb_expect(&bar[b], 16 * slice);
    if (threadIdx.x < 16) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
  }
  if (threadIdx.x == 0 && rank == 0 && blockIdx.x < 16) {
    t[0] = t0;
    t[1] = gtime();
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main() {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  printf("SMs %d\n", nsm);
  // 1. active clusters
  {
    const size_t smem = 200 * 1024;
    CK(cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int cs : {2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(cs * 32);
      cfg.blockDim = dim3(640);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      if (cs == 16) CK(cudaFuncSetAttribute(k_stream, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k_stream, &cfg);
      printf("cluster %2d: max active clusters %d (%d CTAs) %s\n", cs, n, n * cs,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  const size_t total = (size_t)4 << 30;
  char* src;
  CK(cudaMalloc(&src, total));
  CK(cudaMemset(src, 1, total));
  unsigned long long* t;
  CK(cudaMalloc(&t, 4096 * sizeof(unsigned long long)));
  double* sink;
  CK(cudaMalloc(&sink, 64));
  std::vector<unsigned long long> ht(4096);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  // 2. bandwidth vs streaming CTAs (1 CTA per SM, 4 x 32 KB ring)
  {
    const unsigned chunk = 32768;
    CK(cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 7 * chunk));
    for (int depth : {4, 6}) {
      for (int n : {16, 32, 48, 64, 96, 112, 128, 148}) {
        const size_t per = (total / 2 / n) / chunk * chunk;
        float best = 1e9f;
        for (int rep = 0; rep < 5; ++rep) {
          CK(cudaEventRecord(e0));
          k_stream<<<n, 512, depth * chunk>>>(src, per, chunk, depth, depth, 0, t, sink);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          best = ms < best ? ms : best;
        }
        printf("stream depth %d x 32KB, %3d CTAs: %7.1f GB/s (%.1f GB/s per CTA)\n", depth, n,
               per * n / best / 1e6, per / best / 1e6);
      }
    }
    // 3. split: k CTAs with depth 7, the rest depth 3
    for (int k : {16, 32, 64}) {
      const int n = nsm;
      const size_t per = (total / 2 / n) / chunk * chunk;
      k_stream<<<n, 512, 7 * chunk>>>(src, per, chunk, 3, 7, k, t, sink);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(ht.data(), t, 2 * n * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
      double ghi = 0, glo = 0;
      for (int b = 0; b < n; ++b) {
        const double g = per / (double)(ht[2 * b + 1] - ht[2 * b]);
        (b < k ? ghi : glo) += g;
      }
      printf("split: %d CTAs depth 7: %.1f GB/s per CTA; %d CTAs depth 3: %.1f GB/s per CTA\n", k, ghi / k, n - k,
             glo / (n - k));
    }
  }
  // 4. hop chain through global memory
  {
    int* flags;
    double* vec;
    const int H = 2000;
    CK(cudaMalloc(&flags, H * sizeof(int)));
    CK(cudaMalloc(&vec, 2 << 20));
    CK(cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768));
    for (unsigned bytes : {4096u, 28160u}) {
      for (int nchain : {2, 16}) {
        for (int bg : {0, 1}) {
          const int grid = bg ? nsm : nchain;
          const size_t per = (total / nsm) / 32768 * 32768;
          CK(cudaMemset(flags, 0, H * sizeof(int)));
          k_chain<<<grid, 256, 4 * 32768>>>(vec, flags, H, nchain, bytes, src, per, 32768, t, sink);
          CK(cudaDeviceSynchronize());
          CK(cudaMemcpy(ht.data(), t, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
          printf("hop chain: %5u B per hop, %2d chain CTAs, background %s: %.2f us per hop\n", bytes, nchain,
                 bg ? "streaming" : "idle   ", (ht[1] - ht[0]) / 1e3 / H);
        }
      }
    }
  }
  // 5. cluster all-gather
  {
    CK(cudaFuncSetAttribute(k_allgather, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(k_allgather_nb, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (unsigned slice : {256u, 1024u, 1792u, 4096u}) {
      const int rounds = 2000;
      size_t sm = 2 * 16 * slice + slice;
      CK(cudaFuncSetAttribute(k_allgather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      k_allgather<<<16, 256, sm>>>(rounds, slice, t);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(ht.data(), t, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
      printf("cluster16 all-gather (cluster barrier) %5u B slices: %.3f us per round\n", slice,
             (ht[1] - ht[0]) / 1e3 / rounds);
      sm = 4 * 16 * slice + 2 * slice;
      CK(cudaFuncSetAttribute(k_allgather_nb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      k_allgather_nb<<<16, 256, sm>>>(rounds, slice, t);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(ht.data(), t, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
      printf("cluster16 all-gather (mbarrier only)   %5u B slices: %.3f us per round\n", slice,
             (ht[1] - ht[0]) / 1e3 / rounds);
    }
  }
  printf("done\n");
  return 0;
}
