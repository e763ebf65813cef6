// ta_probe.cu — developer probe: tcgen05.mma.cta_group::1.kind::i8 with the A operand in TMEM
// (written by tcgen05.st.32x32b.x32: thread t = row t, 32 columns = the row's 128 K bytes,
// column c holding K bytes 4c..4c+3), B K-major SWIZZLE_128B in shared memory; MMA ks reads A
// columns base + 8ks.  Checked against a CPU integer reference on random data.
// (The comment block below is inherited from sp_probe.cu and describes that probe.)
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


__global__ void k_ta(const uint32_t* a_words, const uint8_t* b, int32_t* d) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
  uint8_t* b_s = sm;
  uint64_t* bar = reinterpret_cast<uint64_t*>(b_s + N * 128);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int t = threadIdx.x, warp = t >> 5;
  if (t < N)
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<uint4*>(b_s + sw128_off(t, j)) = *reinterpret_cast<const uint4*>(b + t * 128 + 16 * j);
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
  const uint32_t A0 = tm + 256;
  const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
  {
    uint32_t w[32];
    for (int i = 0; i < 32; ++i) w[i] = a_words[t * 32 + i];
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(A0 + lane_base),
        "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]),
        "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]),
        "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]),
        "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31]) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (t == 0) {
    const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    for (int ks = 0; ks < 4; ++ks) {
      const uint64_t bd = mdesc(su32(b_s) + 32 * ks, 16, 1024, 2);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm), "r"(A0 + 8 * ks), "l"(bd),
          "r"(idesc), "r"(ks) : "memory");
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

int main() {
  uint32_t* da;
  uint8_t* db;
  int32_t* dd;
  cudaMalloc(&da, 128 * 128);
  cudaMalloc(&db, N * 128);
  cudaMalloc(&dd, 128 * N * 4);
  cudaFuncSetAttribute(k_ta, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  srand(11);
  int fails = 0;
  for (int test = 0; test < 2; ++test) {
    std::vector<uint8_t> A(128 * 128), B(N * 128);
    for (auto& x : B) x = (uint8_t)(rand() & 255);
    for (int r = 0; r < 128; ++r)
      for (int k = 0; k < 128; ++k) A[r * 128 + k] = test == 0 ? (uint8_t)(rand() & 255) : 0;
    if (test == 1)      // one-hot rows: 8 codebooks of 16
      for (int r = 0; r < 128; ++r)
        for (int c = 0; c < 8; ++c) A[r * 128 + 16 * c + rand() % 16] = 1;
    std::vector<int32_t> ref(128 * N, 0);
    for (int r = 0; r < 128; ++r)
      for (int n = 0; n < N; ++n) {
        int32_t s = 0;
        for (int k = 0; k < 128; ++k) s += (int32_t)A[r * 128 + k] * B[n * 128 + k];
        ref[r * N + n] = s;
      }
    cudaMemcpy(da, A.data(), A.size(), cudaMemcpyHostToDevice);   // row r = 32 little-endian words
    cudaMemcpy(db, B.data(), B.size(), cudaMemcpyHostToDevice);
    cudaMemset(dd, 0xff, 128 * N * 4);
    k_ta<<<1, 128, 32768>>>(da, db, dd);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("test %d: CUDA error %s\n", test, cudaGetErrorString(err)); return 2; }
    std::vector<int32_t> got(128 * N);
    cudaMemcpy(got.data(), dd, got.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 128 * N; ++i) bad += got[i] != ref[i];
    printf("test %s: %d / %d mismatches\n", test == 0 ? "random u8" : "one-hot", bad, 128 * N);
    if (bad) printf("  row0: got %d %d %d ref %d %d %d\n", got[0], got[1], got[2], ref[0], ref[1], ref[2]);
    fails += bad != 0;
  }
  printf("%s\n", fails ? "PROBE: MISMATCH" : "PROBE: ALL MATCH");
  return 0;
}
