// sp2_probe.cu — developer probe: semantics of the CTA-pair 2:4-sparse i8 MMA on sm_100a.
//
// One cluster of 2 CTAs.  CTA r holds rows [128r, 128r+128) of a 2:4-sparse A (compressed, K-major
// SWIZZLE_64B, 64 B per row = K 128), their metadata (16 B per row, copied to TMEM by
// tcgen05.cp.cta_group::2.128x128b issued by the leader), and columns [r N/2, (r+1) N/2) of a dense B
// (K-major SWIZZLE_128B).  The leader issues two tcgen05.mma.sp.cta_group::2.kind::i8 (M = 256, K = 64
// each) and commits with a multicast arrive; each CTA then reads its own 128 rows x N accumulators.
// Checked against a CPU integer reference: random 2:4 data and the one-hot pattern of the product.
// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O2 -o sp2_probe sp2_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

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
__host__ __device__ inline uint32_t sw64_off(uint32_t r, uint32_t j) {
  return (r >> 3) * 512u + (r & 7u) * 64u + ((j ^ ((r >> 1) & 3u)) << 4);
}
__host__ __device__ inline uint32_t sw128_off(uint32_t r, uint32_t j) {
  return (r >> 3) * 1024u + (r & 7u) * 128u + ((j ^ (r & 7u)) << 4);
}

// comp: [256][64] compressed A, meta: [256][4] u32, b: [N][128] u8, d: [256][N]
template <int N>
__global__ void __cluster_dims__(2, 1, 1) k_probe(const uint8_t* comp, const uint32_t* meta, const uint8_t* b, int32_t* d) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
  uint8_t* a_s = sm;                    // 8 KB (SW64)
  uint8_t* b_s = sm + 8192;             // N/2 x 128 B (SW128)
  uint8_t* e_s = sm + 8192 + 16384;     // 128 x 16 B metadata
  uint64_t* bar = reinterpret_cast<uint64_t*>(e_s + 2048);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int t = threadIdx.x, warp = t >> 5;
  const int row = 128 * rank + t;
  for (int j = 0; j < 4; ++j)
    *reinterpret_cast<uint4*>(a_s + sw64_off(t, j)) = *reinterpret_cast<const uint4*>(comp + row * 64 + 16 * j);
  if (t < N / 2)
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<uint4*>(b_s + sw128_off(t, j)) = *reinterpret_cast<const uint4*>(b + (rank * (N / 2) + t) * 128 + 16 * j);
  *reinterpret_cast<uint4*>(e_s + 16 * t) = *reinterpret_cast<const uint4*>(meta + 4 * row);
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = *slot;
  const uint32_t E = tm + 448;
  if (rank == 0 && t == 0) {
    const uint32_t idesc = (1u << 2) | (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    const uint64_t ed = mdesc(su32(e_s), 128, 128, 0);
    asm volatile("tcgen05.cp.cta_group::2.128x128b [%0], %1;" ::"r"(E), "l"(ed) : "memory");
    for (int i = 0; i < 2; ++i) {
      const uint64_t ad = mdesc(su32(a_s) + 32 * i, 16, 512, 4);
      const uint64_t bd = mdesc(su32(b_s) + 64 * i, 16, 1024, 2);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
          "tcgen05.mma.sp.cta_group::2.kind::i8 [%0], %1, %2, [%3], %4, p;\n\t}" ::"r"(tm),
          "l"(ad), "l"(bd), "r"(E + 2 * i), "r"(idesc), "r"(i) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(su32(bar)), "h"((uint16_t)3) : "memory");
  }
  __syncwarp();
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
      "@!P1 bra WAIT;\n\t}" ::"r"(su32(bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
  for (int c = 0; c < N; c += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tm + lane_base + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) d[row * N + c + j] = (int32_t)r[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

static bool compress(const std::vector<uint8_t>& A, int rows, std::vector<uint8_t>& comp, std::vector<uint32_t>& meta) {
  comp.assign(rows * 64, 0);
  meta.assign(rows * 4, 0);
  for (int r = 0; r < rows; ++r)
    for (int g = 0; g < 32; ++g) {
      int idx[2] = {0, 0}, n = 0;
      uint8_t val[2] = {0, 0};
      for (int e = 0; e < 4; ++e)
        if (A[r * 128 + 4 * g + e]) {
          if (n == 2) return false;
          idx[n] = e;
          val[n] = A[r * 128 + 4 * g + e];
          ++n;
        }
      if (n == 1) {
        if (idx[0] == 3) { idx[1] = 3; val[1] = val[0]; idx[0] = 0; val[0] = 0; }
        else { idx[1] = 3; val[1] = 0; }
      }
      comp[r * 64 + 2 * g] = val[0];
      comp[r * 64 + 2 * g + 1] = val[1];
      meta[r * 4 + g / 8] |= ((uint32_t)idx[0] | ((uint32_t)idx[1] << 2)) << (4 * (g % 8));
    }
  return true;
}

template <int N>
static int run() {
  uint8_t *dc, *db;
  uint32_t* dm;
  int32_t* dd;
  cudaMalloc(&dc, 256 * 64);
  cudaMalloc(&dm, 256 * 16);
  cudaMalloc(&db, N * 128);
  cudaMalloc(&dd, 256 * N * 4);
  cudaFuncSetAttribute(k_probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40960);
  int fails = 0;
  for (int test = 0; test < 2; ++test) {
    std::vector<uint8_t> A(256 * 128, 0), B(N * 128);
    for (auto& x : B) x = (uint8_t)(rand() & 255);
    for (int r = 0; r < 256; ++r) {
      if (test == 0) {
        for (int g = 0; g < 32; ++g) {
          const int pat = rand() % 4;
          int e0 = rand() % 4, e1 = rand() % 4;
          if (pat >= 1) A[r * 128 + 4 * g + e0] = (uint8_t)(1 + rand() % 255);
          if (pat >= 2 && e1 != e0) A[r * 128 + 4 * g + e1] = (uint8_t)(1 + rand() % 255);
        }
      } else {
        for (int c = 0; c < 8; ++c) A[r * 128 + 16 * c + rand() % 16] = 1;
      }
    }
    std::vector<uint8_t> comp;
    std::vector<uint32_t> meta;
    if (!compress(A, 256, comp, meta)) { printf("compress failed\n"); return 1; }
    std::vector<int32_t> ref(256 * N, 0);
    for (int r = 0; r < 256; ++r)
      for (int n = 0; n < N; ++n) {
        int32_t s = 0;
        for (int k = 0; k < 128; ++k) s += (int32_t)A[r * 128 + k] * B[n * 128 + k];
        ref[r * N + n] = s;
      }
    cudaMemcpy(dc, comp.data(), comp.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dm, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, B.data(), B.size(), cudaMemcpyHostToDevice);
    cudaMemset(dd, 0xff, 256 * N * 4);
    k_probe<N><<<2, 128, 40960>>>(dc, dm, db, dd);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("N=%d test %d: CUDA error %s\n", N, test, cudaGetErrorString(err)); return 2; }
    std::vector<int32_t> got(256 * N);
    cudaMemcpy(got.data(), dd, got.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0, bad0 = 0, bad1 = 0;
    for (int i = 0; i < 256 * N; ++i)
      if (got[i] != ref[i]) { ++bad; (i / N < 128 ? bad0 : bad1)++; }
    printf("N=%d test %-8s: %d / %d mismatches (rows of CTA0 %d, CTA1 %d)\n", N, test ? "onehot" : "random", bad, 256 * N, bad0, bad1);
    if (bad) printf("  e.g. row 0: got %d %d ref %d %d; row 128: got %d ref %d\n", got[0], got[1], ref[0], ref[1], got[128 * N], ref[128 * N]);
    fails += bad != 0;
  }
  return fails;
}

int main() {
  srand(11);
  int fails = run<256>() + run<224>() + run<128>();
  printf("%s\n", fails ? "PROBE: MISMATCH" : "PROBE: ALL MATCH");
  return 0;
}
