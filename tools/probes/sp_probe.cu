// sp_probe.cu — developer probe: semantics of tcgen05.mma.sp.cta_group::1.kind::i8 on sm_100a.
//
// Checks (against a CPU integer reference) one 128-row CTA tile: D[128][N] = A[128][128] . B[N][128]^T
// with A 2:4 sparse, stored compressed (2 of every 4 K-elements, 64 B per row) in a K-major
// SWIZZLE_64B tile, B dense K-major SWIZZLE_128B, two sparse MMAs of K = 64 each.  The sparse
// metadata (per group of 4 K-elements: bits[1:0] = logical index of stored element 0, bits[3:2] of
// element 1; group g of an MMA at nibble g of the row's 64-bit word) reaches TMEM three ways:
//   mode 0: tcgen05.st from registers, MMA i reads columns E + 2i
//   mode 1: tcgen05.st, MMA i reads columns E + 4i
//   mode 2: tcgen05.cp.128x128b from shared memory (16 B per row), MMA i reads E + 2i
// Test 0 is diagnostic (row r has one nonzero at K = r, B[0][k] = k + 1, so D[r][0] - 1 is the K the
// hardware used); test 1 is random 2:4 data; test 2 is the one-hot pattern the product uses.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o sp_probe sp_probe.cu
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

// comp: [128][64] compressed A (row-major), meta: [128][4] u32 (K-block metadata), b: [N][128] u8
__global__ void k_probe(const uint8_t* comp, const uint32_t* meta, const uint8_t* b, int32_t* d, int mode) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
  uint8_t* a_s = sm;                 // 8 KB (SW64)
  uint8_t* b_s = sm + 8192;          // N x 128 B (SW128)
  uint8_t* e_s = b_s + N * 128;      // 128 x 16 B metadata (mode 2)
  uint64_t* bar = reinterpret_cast<uint64_t*>(e_s + 2048);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int t = threadIdx.x, warp = t >> 5;
  for (int j = 0; j < 4; ++j)
    *reinterpret_cast<uint4*>(a_s + sw64_off(t, j)) = *reinterpret_cast<const uint4*>(comp + t * 64 + 16 * j);
  if (t < N)
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<uint4*>(b_s + sw128_off(t, j)) = *reinterpret_cast<const uint4*>(b + t * 128 + 16 * j);
  *reinterpret_cast<uint4*>(e_s + 16 * t) = *reinterpret_cast<const uint4*>(meta + 4 * t);
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
  const uint32_t E = tm + 256;
  const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
  if (mode == 0) {
    const uint32_t* m = meta + 4 * t;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(E + lane_base), "r"(m[0]),
                 "r"(m[1]), "r"(m[2]), "r"(m[3]) : "memory");
  } else if (mode == 1) {
    const uint32_t* m = meta + 4 * t;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(E + lane_base),
                 "r"(m[0]), "r"(m[1]), "r"(0u), "r"(0u), "r"(m[2]), "r"(m[3]), "r"(0u), "r"(0u) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (t == 0) {
    const uint32_t idesc = (1u << 2) | (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (mode == 2) {
      const uint64_t ed = mdesc(su32(e_s), 128, 128, 0);
      asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(E), "l"(ed) : "memory");
    }
    for (int i = 0; i < 2; ++i) {
      const uint64_t ad = mdesc(su32(a_s) + 32 * i, 16, 512, 4);
      const uint64_t bd = mdesc(su32(b_s) + 64 * i, 16, 1024, 2);
      const uint32_t e = E + (uint32_t)(mode == 1 ? 4 * i : 2 * i);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
          "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%3], %4, p;\n\t}" ::"r"(tm),
          "l"(ad), "l"(bd), "r"(e), "r"(idesc), "r"(i) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
  }
  __syncwarp();
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
      "@!P1 bra WAIT;\n\t}" ::"r"(su32(bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c = 0; c < N; c += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tm + lane_base + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) d[t * N + c + j] = (int32_t)r[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

// Compress a 2:4-sparse row-major A[128][128] into comp[128][64] + meta[128][4]
// (stored pair per group: ascending logical indices; one nonzero -> (i, 3) or (0, 3) as below).
static bool compress(const std::vector<uint8_t>& A, std::vector<uint8_t>& comp, std::vector<uint32_t>& meta) {
  comp.assign(128 * 64, 0);
  meta.assign(128 * 4, 0);
  for (int r = 0; r < 128; ++r)
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
      const uint32_t nib = (uint32_t)idx[0] | ((uint32_t)idx[1] << 2);
      meta[r * 4 + g / 8] |= nib << (4 * (g % 8));
    }
  return true;
}

int main() {
  const char* tname[3] = {"diag", "random2:4", "onehot"};
  uint8_t *dc, *db;
  uint32_t* dm;
  int32_t* dd;
  cudaMalloc(&dc, 128 * 64);
  cudaMalloc(&dm, 128 * 16);
  cudaMalloc(&db, N * 128);
  cudaMalloc(&dd, 128 * N * 4);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  srand(7);
  int fails = 0;
  for (int test = 0; test < 3; ++test) {
    std::vector<uint8_t> A(128 * 128, 0), B(N * 128);
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < 128; ++k) B[n * 128 + k] = (uint8_t)(test == 0 && n == 0 ? k + 1 : rand() & 255);
    for (int r = 0; r < 128; ++r) {
      if (test == 0) {
        A[r * 128 + r] = 1;
      } else if (test == 1) {
        for (int g = 0; g < 32; ++g) {
          const int pat = rand() % 4;           // 0: none, 1: one, 2/3: two nonzeros
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
    if (!compress(A, comp, meta)) { printf("compress failed\n"); return 1; }
    std::vector<int32_t> ref(128 * N, 0);
    for (int r = 0; r < 128; ++r)
      for (int n = 0; n < N; ++n) {
        int32_t s = 0;
        for (int k = 0; k < 128; ++k) s += (int32_t)A[r * 128 + k] * B[n * 128 + k];
        ref[r * N + n] = s;
      }
    cudaMemcpy(dc, comp.data(), comp.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dm, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, B.data(), B.size(), cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 3; ++mode) {
      cudaMemset(dd, 0xff, 128 * N * 4);
      k_probe<<<1, 128, 32768>>>(dc, dm, db, dd, mode);
      cudaError_t err = cudaDeviceSynchronize();
      if (err != cudaSuccess) { printf("test %s mode %d: CUDA error %s\n", tname[test], mode, cudaGetErrorString(err)); return 2; }
      std::vector<int32_t> got(128 * N);
      cudaMemcpy(got.data(), dd, got.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int i = 0; i < 128 * N; ++i) bad += got[i] != ref[i];
      printf("test %-10s mode %d: %d / %d mismatches\n", tname[test], mode, bad, 128 * N);
      if (bad && test == 0) {
        printf("  hw K per row (D[r][0]-1):");
        for (int r = 0; r < 128; ++r) printf(" %d", got[r * N] - 1);
        printf("\n");
      }
      fails += bad != 0;
    }
  }
  printf("%s\n", fails ? "PROBE: MISMATCH" : "PROBE: ALL MATCH");
  return 0;
}
