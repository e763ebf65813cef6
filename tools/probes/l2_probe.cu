// l2_probe.cu — developer probe: L2 -> shared-memory bulk-copy bandwidth on B200 (the LUT
// streaming of the streamed-LUT TC mode), with and without cluster multicast.
//   k_l2  : one CTA per SM, S stages x B bytes, chunks of an L2-resident buffer (or an HBM-sized one)
//   k_mc  : clusters of CS CTAs; CTA rank r issues chunks r, r+CS, ... of each round with
//           .multicast::cluster to every CTA of the cluster (one L2 read feeds CS SMs); a cluster
//           barrier per round of S stages frees the ring.
// Delivered bandwidth = bytes landed in shared memory (all CTAs) / time.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_probe l2_probe.cu
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_par(uint64_t* bar, uint32_t par) {
  asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(su32(bar)),
               "r"(par) : "memory");
}

__global__ void k_l2(const char* src, size_t nchunks, int B, int S, int per_cta, unsigned long long* sink) {
  extern __shared__ __align__(1024) char sm[];
  uint64_t* bar = (uint64_t*)(sm + (size_t)S * B);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + s)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  auto issue = [&](int k, int s) {
    const size_t t = ((size_t)blockIdx.x * 7919 + (size_t)k) % nchunks;
    asm volatile("{.reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;}" ::"r"(su32(bar + s)), "r"(B) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(sm + (size_t)s * B)), "l"(src + t * B), "r"(B), "r"(su32(bar + s)) : "memory");
  };
  for (int k = 0; k < S && k < per_cta; ++k) issue(k, k);
  unsigned acc = 0;
  for (int k = 0; k < per_cta; ++k) {
    const int s = k % S;
    wait_par(bar + s, (k / S) & 1);
    acc += sm[(size_t)s * B];
    if (k + S < per_cta) issue(k + S, s);
  }
  if (acc == 0x12345678) sink[0] = acc;
}

__global__ void k_mc(const char* src, size_t nchunks, int B, int S, int rounds, unsigned long long* sink) {
  extern __shared__ __align__(1024) char sm[];
  uint64_t* bar = (uint64_t*)(sm + (size_t)S * B);
  uint32_t rank, cs;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(cs));
  uint32_t cid;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + s)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  const uint16_t mask = (uint16_t)((1u << cs) - 1);
  unsigned acc = 0;
  for (int r = 0; r < rounds; ++r) {
    if (threadIdx.x == 0) {
      for (int s = 0; s < S; ++s)
        asm volatile("{.reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;}" ::"r"(su32(bar + s)), "r"(B) : "memory");
    }
    // every CTA's expect_tx is posted before any multicast of this round can complete on it
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0) {
      for (int s = (int)rank; s < S; s += (int)cs) {
        const size_t t = ((size_t)cid * 7919 + (size_t)r * S + s) % nchunks;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
            ::"r"(su32(sm + (size_t)s * B)), "l"(src + t * B), "r"(B), "r"(su32(bar + s)), "h"(mask) : "memory");
      }
      for (int s = 0; s < S; ++s) {
        wait_par(bar + s, r & 1);
        acc += sm[(size_t)s * B];
      }
    }
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  if (acc == 0x12345678) sink[0] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t big = (size_t)1 << 30;
  char* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(k_l2, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k_mc, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k_mc, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t l2buf = (size_t)16 << 20;
  for (size_t span : {l2buf, (size_t)4 << 20, big}) {
    for (int B : {16384, 32768}) {
      for (int S : {2, 4, 6}) {
        const int per_cta = 2000;
        const size_t nchunks = span / B;
        auto run = [&] { k_l2<<<sms, 32, (size_t)S * B + 64>>>(buf, nchunks, B, S, per_cta, sink); };
        run();
        cudaEventRecord(a);
        for (int i = 0; i < 3; ++i) run();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = 3.0 * sms * per_cta * (double)B;
        printf("{\"probe\": \"l2\", \"span_MB\": %zu, \"B\": %d, \"S\": %d, \"TBps\": %.2f, \"GBps_per_sm\": %.1f}\n",
               span >> 20, B, S, bytes / (ms * 1e-3) / 1e12, bytes / (ms * 1e-3) / 1e9 / sms);
      }
    }
  }
  for (int cs : {1, 2, 4}) {
    for (int S : {4, 6}) {
      const int B = 32768, rounds = 400;
      const size_t nchunks = l2buf / B;
      const int grid = sms / cs * cs;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(32);
      cfg.dynamicSmemBytes = (size_t)S * B + 64;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      auto run = [&] { return cudaLaunchKernelEx(&cfg, k_mc, (const char*)buf, nchunks, B, S, rounds, sink); };
      cudaError_t e = run();
      cudaDeviceSynchronize();
      if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("{\"probe\": \"mc\", \"cs\": %d, \"error\": \"%s\"}\n", cs, cudaGetErrorString(e)); continue; }
      cudaEventRecord(a);
      for (int i = 0; i < 3; ++i) run();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double delivered = 3.0 * grid * rounds * S * (double)B;
      printf("{\"probe\": \"mc\", \"cs\": %d, \"B\": %d, \"S\": %d, \"delivered_TBps\": %.2f, \"l2_read_TBps\": %.2f, \"GBps_per_sm\": %.1f}\n",
             cs, B, S, delivered / (ms * 1e-3) / 1e12, delivered / cs / (ms * 1e-3) / 1e12,
             delivered / (ms * 1e-3) / 1e9 / grid);
    }
  }
  return 0;
}
