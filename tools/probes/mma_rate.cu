// mma_rate.cu — developer probe: tcgen05.mma issue rate on sm_100a.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

constexpr int N = 64;   // UMMA N
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t mdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__host__ __device__ inline uint32_t sw64_off(uint32_t r, uint32_t j) {   // 16-B chunk j (0..3) of row r
  return (r >> 3) * 512u + (r & 7u) * 64u + ((j ^ ((r >> 1) & 3u)) << 4);
}
__host__ __device__ inline uint32_t sw128_off(uint32_t r, uint32_t j) {
  return (r >> 3) * 1024u + (r & 7u) * 128u + ((j ^ (r & 7u)) << 4);
}


// mma_rate: back-to-back tcgen05.mma (one CTA per SM, one issuing thread), operands in shared
// memory (SWIZZLE_128B K-major; contents irrelevant), or A in TMEM; accumulate into TMEM.
// kind 0: i8 (K=32/instr), kind 1: f16 (bf16 inputs, K=16/instr), kind 2: i8 with A in TMEM,
// kind 3: i8 sparse (K=64/instr).  Reports ns per instruction and the implied dense TOPS.
__global__ void k_rate(int kind, int n, int iters, unsigned long long* out, int commit_every) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
  uint8_t* a_s = sm;                 // 128 x 128 B
  uint8_t* b_s = sm + 16384;         // 256 x 128 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 16384 + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 4);
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < (16384 + 32768) / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x01010101u, 0, 0, 0);
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = *slot;
  if (t == 0) {
    uint32_t idesc;
    if (kind == 1) idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);  // f32 acc, bf16 A/B
    else idesc = (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24) | (kind == 3 ? 4u : 0u);
    const uint64_t ad = mdesc(su32(a_s), 16, 1024, 2), bd = mdesc(su32(b_s), 16, 1024, 2);
    const uint64_t ad64 = mdesc(su32(a_s), 16, 512, 4);
    uint64_t* bar2 = bar + 2;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t acc = i > 0;
      if (commit_every && (i & (commit_every - 1)) == 0 && i > 0)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar2)) : "memory");
      if (kind == 0 || kind == 1) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(ad + 2 * (i & 3)), "l"(bd + 2 * (i & 3)), "r"(idesc), "r"(acc) : "memory");
      } else if (kind == 2) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm), "r"(tm + 256 + 8 * (i & 3)), "l"(bd + 2 * (i & 3)), "r"(idesc), "r"(acc) : "memory");
      } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
                     "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%3], %4, p;\n\t}" ::"r"(tm), "l"(ad64 + 2 * (i & 1)), "l"(bd + 4 * (i & 1)), "r"(tm + 480), "r"(idesc), "r"(acc) : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
    asm volatile("{\n\t.reg .pred P1;\n\tWAIT:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra WAIT;\n\t}" ::"r"(su32(bar)) : "memory");
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned long long* dout;
  cudaMalloc(&dout, 8);
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[4] = {"i8_ss", "bf16_ss", "i8_ts(A in TMEM)", "i8_sparse_ss"};
  for (int kind : {0})
    for (int n : {256}) for (int ce : {0, 4, 8, 16}) {
      const int iters = 20000;
      k_rate<<<sms, 128, 64 * 1024>>>(kind, n, 100, dout, ce);
      cudaEventRecord(a);
      k_rate<<<sms, 128, 64 * 1024>>>(kind, n, iters, dout, ce);
      cudaEventRecord(b);
      cudaError_t e = cudaEventSynchronize(b);
      if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("{\"kind\": \"%s\", \"n\": %d, \"error\": \"%s\"}\n", names[kind], n, cudaGetErrorString(e)); return 1; }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      unsigned long long cyc;
      cudaMemcpy(&cyc, dout, 8, cudaMemcpyDeviceToHost);
      const double kk = kind == 1 ? 16 : (kind == 3 ? 64 : 32);
      const double ops = 2.0 * 128 * n * kk * iters * sms;
      printf("{\"commit_every\": %d, \"kind\": \"%s\", \"n\": %d, \"ns_per_mma\": %.1f, \"cycles_per_mma\": %.1f, \"dense_equiv_TOPS\": %.0f}\n", ce, names[kind], n,
             ms * 1e6 / iters, (double)cyc / iters, ops / (ms * 1e-3) / 1e12);
    }
  return 0;
}
