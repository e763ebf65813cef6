// smem_contention.cu — developer probe: does shared-memory traffic from other roles slow the
// tcgen05 i8 MMA, and does cta_group::2 halve the per-SM operand traffic?
//
// One cluster of `cg` CTAs per SM pair (or one CTA per SM for cg = 1).  The MMA thread (leader CTA)
// issues `iters` back-to-back tcgen05.mma kind::i8 (dense K=32 or 2:4-sparse K=64; M = 128 per CTA,
// N = 256 total) from shared memory.  Meanwhile, optionally:
//   sts_warps warps write 16-byte chunks (conflict-free, 8 STS.128 per loop) into a scratch region,
//   one thread keeps `tma_inflight` 32 KB bulk copies (L2-resident source) landing in shared memory.
// Reports cycles per MMA and the bytes per cycle the other roles achieved while it ran.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t mdesc(uint32_t saddr, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  for (uint32_t it = 0; !mbar_try(b, ph); ++it)
    if (it > (1u << 26)) __trap();
}

struct Res { unsigned long long mma_cyc, sts_bytes, tma_bytes; };

// smem: A 16 KB | B 32 KB | STS scratch 32 KB | TMA dst 4 x 32 KB | bars
template <int cg, int sparse>
__global__ void k_probe(int sparse_unused, int n, int iters, int sts_warps, int tma_inflight, int kmask,
                        const uint8_t* src, Res* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
  uint8_t* a_s = sm;
  uint8_t* b_s = sm + 16384;
  uint8_t* sts_s = sm + 49152;
  uint8_t* tma_s = sm + 81920;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 81920 + 4 * 32768);
  volatile uint32_t* done = reinterpret_cast<volatile uint32_t*>(bar + 8);
  uint32_t* slot = const_cast<uint32_t*>(done + 1);
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(bar + 10);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const uint32_t rank = cg == 2 ? cluster_rank() : 0;
  for (int i = t; i < 49152 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x01010101u, 0, 0, 0);
  if (t == 0) {
    for (int i = 0; i < 6; ++i) mbar_init(bar + i, 1);
    *done = 0;
    cnt[0] = cnt[1] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    if constexpr (cg == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(slot)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(slot)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if constexpr (cg == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = *slot;
  if (warp == 0) {
    // ------------------------------------------------ MMA issuer (leader) / waiter (peer)
    if (lane == 0) {
      unsigned long long t0 = clock64();
      if (rank == 0) {
        const uint32_t m = cg == 2 ? 256 : 128;
        const uint32_t idesc = (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((m >> 4) << 24) | (sparse ? 4u : 0u);
        const uint64_t ad = sparse != 0 ? mdesc(su32(a_s), 512, 4) : mdesc(su32(a_s), 1024, 2);
        const uint64_t bd = mdesc(su32(b_s), 1024, 2);
        for (int i = 0; i < iters; ++i) {
          const uint32_t acc = i > 0;
          const uint64_t a = ad + 2 * (i & kmask), b = bd + (sparse ? 4 : 2) * (i & kmask);
          if constexpr (cg == 2) {
            if constexpr (sparse != 0)
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
                           "tcgen05.mma.sp.cta_group::2.kind::i8 [%0], %1, %2, [%3], %4, p;\n\t}" ::"r"(tm), "l"(a), "l"(b),
                           "r"(tm + 480), "r"(idesc), "r"(acc) : "memory");
            else
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(a), "l"(b), "r"(idesc),
                           "r"(acc) : "memory");
          } else {
            if constexpr (sparse != 0)
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
                           "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%3], %4, p;\n\t}" ::"r"(tm), "l"(a), "l"(b),
                           "r"(tm + 480), "r"(idesc), "r"(acc) : "memory");
            else
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(a), "l"(b), "r"(idesc),
                           "r"(acc) : "memory");
          }
        }
        if constexpr (cg == 2)
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                       ::"r"(su32(bar)), "h"((uint16_t)3) : "memory");
        else
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
      }
      mbar_wait(bar, 0);
      unsigned long long t1 = clock64();
      *done = 1;
      if (blockIdx.x == 0) out->mma_cyc = t1 - t0;
    }
  } else if (warp == 1) {
    // ------------------------------------------------ TMA bulk copies (L2-resident 1 MB source)
    if (lane == 0 && tma_inflight > 0) {
      unsigned long long bytes = 0;
      int k = 0;
      uint32_t ph[4] = {0, 0, 0, 0};
      bool busy[4] = {false, false, false, false};
      auto issue = [&](int s) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + 1 + s)), "r"(32768) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(tma_s + s * 32768)), "l"(src + (size_t)(k & 31) * 32768), "r"(32768), "r"(su32(bar + 1 + s)) : "memory");
        busy[s] = true;
        ++k;
      };
      for (int s = 0; s < tma_inflight; ++s) issue(s);
      while (!*done) {
        for (int s = 0; s < tma_inflight && !*done; ++s) {
          mbar_wait(bar + 1 + s, ph[s]);
          ph[s] ^= 1;
          busy[s] = false;
          bytes += 32768;
          issue(s);
        }
      }
      for (int s = 0; s < tma_inflight; ++s)
        if (busy[s]) mbar_wait(bar + 1 + s, ph[s]);   // drain outstanding copies
      if (blockIdx.x == 0) out->tma_bytes = bytes;
    }
  } else if (warp >= 2 && warp < 2 + sts_warps) {
    // ------------------------------------------------ STS.128 writers, conflict-free
    const int w = warp - 2;
    unsigned long long loops = 0;
    uint4 v = make_uint4(t, 1, 2, 3);
    uint8_t* base = sts_s + w * 4096 + lane * 16;
    while (!*done) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(su32(base + j * 512)), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
      ++loops;
    }
    if (blockIdx.x == 0 && lane == 0) atomicAdd(&cnt[0], loops * 8 * 512);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (blockIdx.x == 0 && t == 0) out->sts_bytes = cnt[0];
  if constexpr (cg == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    if constexpr (cg == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  Res* dres;
  cudaMalloc(&dres, sizeof(Res));
  uint8_t* src;
  cudaMalloc(&src, 1 << 20);
  cudaMemset(src, 1, 1 << 20);
  const size_t smem = 81920 + 4 * 32768 + 1024 + 256;
  cudaFuncSetAttribute(k_probe<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_probe<2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_probe<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_probe<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int combos[4][2] = {{0, 0}, {4, 0}, {0, 2}, {4, 2}};
  for (int cg : {1, 2})
    for (int sparse : {0, 1})
      for (int n : {128, 256})
        for (int km : {1, 3})
        for (auto& cb : combos) {
          if (km == 3 && (sparse || cb[0] || cb[1])) continue;
          const int sts = cb[0], tma = cb[1];
          const int iters = 20000;
          cudaLaunchConfig_t cfg{};
          cfg.gridDim = dim3(sms / 2 * 2);
          cfg.blockDim = dim3(32 * 10);
          cfg.dynamicSmemBytes = smem;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = cg;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = cg == 2 ? 1 : 0;
          cudaMemset(dres, 0, sizeof(Res));
          auto kern = cg == 2 ? (sparse ? k_probe<2, 1> : k_probe<2, 0>) : (sparse ? k_probe<1, 1> : k_probe<1, 0>);
          const int kmask = sparse ? 1 : km;
          cudaError_t e = cudaLaunchKernelEx(&cfg, kern, sparse, n, 200, sts, tma, kmask, (const uint8_t*)src, dres);
          if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, kern, sparse, n, iters, sts, tma, kmask, (const uint8_t*)src, dres);
          if (e == cudaSuccess) e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("{\"cg\": %d, \"sparse\": %d, \"error\": \"%s\"}\n", cg, sparse, cudaGetErrorString(e)); return 1; }
          Res r;
          cudaMemcpy(&r, dres, sizeof r, cudaMemcpyDeviceToHost);
          const double cyc = (double)r.mma_cyc;
          printf("{\"cg\": %d, \"kmask\": %d, \"sparse\": %d, \"n\": %d, \"sts_warps\": %d, \"tma_inflight\": %d, \"cycles_per_mma\": %.1f, "
                 "\"sts_B_per_cyc\": %.1f, \"tma_B_per_cyc\": %.1f}\n",
                 cg, kmask, sparse, n, sts, tma, cyc / iters, r.sts_bytes / cyc, r.tma_bytes / cyc);
        }
  return 0;
}
