// Microbenchmark: read-streaming bandwidth on B200 with (a) cp.async.bulk (TMA, UBLKCP) rings of
// S stages x B bytes per CTA, one CTA per SM; (b) plain LDG.128 grid-stride; (c) STG.128 writes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_bulk(const char* src, size_t total, int B, int S, unsigned long long* sink) {
  extern __shared__ __align__(16) char sm[];
  uint64_t* bar = (uint64_t*)(sm + (size_t)S * B);
  const size_t ntiles = total / B;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + s)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](size_t t, int s) {
    asm volatile("{.reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;}" ::"r"(su32(bar + s)), "r"(B) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(sm + (size_t)s * B)), "l"(src + t * B), "r"(B), "r"(su32(bar + s)) : "memory");
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < S; ++k) { size_t t = blockIdx.x + (size_t)k * gridDim.x; if (t < ntiles) issue(t, k); }
  unsigned acc = 0;
  int k = 0;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = k % S;
    const uint32_t par = (k / S) & 1;
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(su32(bar + s)), "r"(par) : "memory");
    acc += sm[(size_t)s * B + threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) { size_t nt = t + (size_t)S * gridDim.x; if (nt < ntiles) issue(nt, s); }
  }
  if (acc == 0x12345678) sink[0] = acc;
}

__global__ void k_ldg(const uint4* src, size_t n, unsigned long long* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(src + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) sink[0] = acc;
}

__global__ void k_ldg_unroll(const uint4* src, size_t n, unsigned long long* sink) {
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n; i += stride) { uint4 v = __ldcs(src + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345678) sink[0] = acc;
}

__global__ void k_stg(uint4* dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(dst + i, make_uint4(i, 1, 2, 3));
}


// Emulates the TC epilogue's store pattern: out is N x ldo fp32; CTA = (group, slice of NS cols);
// per 128-row tile, warp (q, h) of W warps writes rows 32q..32q+31, 32-col chunks j0 = 32h' + 32*nh*i,
// each STG.128 instruction = 4 rows x 128 B.
__global__ void k_stg_tile(float* out, int64_t N, int ldo, int NS, int G, int nh) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, h = warp >> 2;
  const int slice = blockIdx.x % G, group = blockIdx.x / G, ngroups = gridDim.x / G;
  const int64_t ntiles = (N + 127) / 128;
  const int cq = lane & 7, rsub = lane >> 3;
  for (int64_t tile = group; tile < ntiles; tile += ngroups) {
    const int64_t row0 = tile * 128 + q * 32;
    for (int j0 = h * 32; j0 < NS; j0 += 32 * nh) {
      float* o = out + (row0 + rsub) * ldo + slice * NS + j0 + 4 * cq;
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        if (row0 + it * 4 + rsub < N) __stcs(reinterpret_cast<float4*>(o), make_float4(1.f, 2.f, 3.f, (float)it));
        o += 4 * ldo;
      }
    }
  }
}


// Mixed traffic: CTAs [0, Er) stream-read `rd` bytes with bulk copies (B-byte stages, S deep);
// the others write `wr` bytes with STG.128.  Returns when both are done.
__global__ void k_mixed(const char* src, size_t rd, uint4* dst, size_t wr_n16, int B, int S, int Er,
                        unsigned long long* sink) {
  extern __shared__ __align__(16) char sm[];
  if ((int)blockIdx.x < Er) {
    uint64_t* bar = (uint64_t*)(sm + (size_t)S * B);
    const size_t ntiles = rd / B;
    if (threadIdx.x == 0) {
      for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + s)));
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    auto issue = [&](size_t t, int s) {
      asm volatile("{.reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;}" ::"r"(su32(bar + s)), "r"(B) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(sm + (size_t)s * B)), "l"(src + t * B), "r"(B), "r"(su32(bar + s)) : "memory");
    };
    if (threadIdx.x == 0)
      for (int k = 0; k < S; ++k) { size_t t = blockIdx.x + (size_t)k * Er; if (t < ntiles) issue(t, k); }
    unsigned acc = 0;
    int k = 0;
    for (size_t t = blockIdx.x; t < ntiles; t += Er, ++k) {
      const int s = k % S;
      const uint32_t par = (k / S) & 1;
      asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(su32(bar + s)), "r"(par) : "memory");
      acc += sm[(size_t)s * B + threadIdx.x];
      __syncthreads();
      if (threadIdx.x == 0) { size_t nt = t + (size_t)S * Er; if (nt < ntiles) issue(nt, s); }
    }
    if (acc == 0x12345678) sink[0] = acc;
  } else {
    const int nw = gridDim.x - Er;
    for (size_t i = (blockIdx.x - Er) * (size_t)blockDim.x + threadIdx.x; i < wr_n16; i += (size_t)nw * blockDim.x)
      __stcs(dst + i, make_uint4(i, 1, 2, 3));
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = (size_t)188 * 3136 * 320;   // ~188 MB (60000 rows of 3136 B, padded)
  char* buf; cudaMalloc(&buf, total * 2);
  char* buf2 = buf + total;
  cudaMemset(buf, 1, total * 2);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto time = [&](auto fn) {
    for (int i = 0; i < 3; ++i) { fn(i); }
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    const int it = 20;
    for (int i = 0; i < it; ++i) fn(i);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / it;
  };
  // alternate two buffers so L2 never holds the next input
  for (int B : {8192, 16384, 32768, 65536}) for (int S : {2, 3, 4, 6, 8, 12}) {
    if ((size_t)S * B + 128 > 220 * 1024) continue;
    for (int cps : {1, 2}) {
      float ms = time([&](int i) { k_bulk<<<sms * cps, 128, S * B + 128>>>((i & 1) ? buf2 : buf, total - total % B, B, S, sink); });
      if (cps == 2 && 2 * ((size_t)S * B + 128) > 228 * 1024) continue;
      printf("{\"kind\":\"bulk\",\"B\":%d,\"S\":%d,\"ctas_per_sm\":%d,\"GBps\":%.1f}\n", B, S, cps, total / (ms * 1e-3) / 1e9);
    }
  }
  for (int tpb : {256, 512, 1024}) for (int bpsm : {1, 2, 4, 8}) {
    if (tpb * bpsm > 2048) continue;
    float ms = time([&](int i) { k_ldg<<<sms * bpsm, tpb>>>((const uint4*)((i & 1) ? buf2 : buf), total / 16, sink); });
    float ms2 = time([&](int i) { k_ldg_unroll<<<sms * bpsm, tpb>>>((const uint4*)((i & 1) ? buf2 : buf), total / 16, sink); });
    printf("{\"kind\":\"ldg\",\"tpb\":%d,\"bpsm\":%d,\"GBps\":%.1f,\"GBps_unroll8\":%.1f}\n", tpb, bpsm, total / (ms * 1e-3) / 1e9, total / (ms2 * 1e-3) / 1e9);
  }
  for (int tpb : {256, 1024}) for (int bpsm : {1, 2, 8}) {
    if (tpb * bpsm > 2048) continue;
    float ms = time([&](int i) { k_stg<<<sms * bpsm, tpb>>>((uint4*)((i & 1) ? buf2 : buf), total / 16); });
    printf("{\"kind\":\"stg\",\"tpb\":%d,\"bpsm\":%d,\"GBps\":%.1f}\n", tpb, bpsm, total / (ms * 1e-3) / 1e9);
  }
  {
    const int64_t N = 60000; const int ldo = 512;
    for (int G : {1, 2, 4}) for (int nh : {1, 2, 4}) for (int ctas : {1, 2}) {
      const int NS = 512 / G;
      const int grid = G * ((sms * ctas) / G);
      float ms = time([&](int i) { k_stg_tile<<<grid, 128 * nh>>>((float*)((i & 1) ? buf2 : buf), N, ldo, NS, G, nh); });
      printf("{\"kind\":\"stg_tile\",\"G\":%d,\"warps\":%d,\"ctas_per_sm\":%d,\"GBps\":%.1f}\n", G, 4 * nh, ctas, N * ldo * 4.0 / (ms * 1e-3) / 1e9);
    }
  }
  {
    cudaFuncSetAttribute(k_mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    const size_t rd = (size_t)60000 * 3136, wr = (size_t)60000 * 2048;
    for (int Er : {60, 74, 88, 100, 148}) {
      float ms = time([&](int i) { k_mixed<<<(Er == 148 ? 296 : sms), 256, 4 * 25088 + 128>>>((i & 1) ? buf2 : buf, rd - rd % 25088, (uint4*)((i & 1) ? buf : buf2), wr / 16, 25088, 4, Er == 148 ? 148 : Er, sink); });
      printf("{\"kind\":\"mixed\",\"read_ctas\":%d,\"us\":%.1f,\"GBps_total\":%.1f}\n", Er, ms * 1e3, (rd + wr) / (ms * 1e-3) / 1e9);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"status\":\"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
