// common.cuh — device helpers shared by the ITLUMM kernels (sm_100a only).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "itlumm kernels are written for sm_100a (B200) only"
#endif

namespace itlumm {

constexpr int kLevels = 4;   // "exactly 4 comparisons"
constexpr int kK = 16;       // prototypes per codebook

// Device-side view of a plan (passed by value to kernels).
struct DevPlan {
  const int32_t* cols;    // [C][4] absolute gather column: perm[b_c + split_dim[c][t]] (a1 folded)
  const float* thr_t;     // [15][C] thresholds, heap index major (lanes = codebooks -> no bank conflicts)
  const uint8_t* lut;     // [C][16][Mp] uint8 LUT, Mp = roundup(M,16), zero padded
  const float* scale;     // [Mp]
  const float* offtot;    // [Mp] (float)((double)C*lo + bias)
  const float* offavg;    // [Mp] avg16 summation: (float)((double)C*lo + bias - 16*(C/16)*(double)scale)
  int D, C, M, Mp;
};

template <typename T> struct InTraits;
template <> struct InTraits<float> {
  static __device__ __forceinline__ float load(const float* p) { return __ldg(p); }
  static __device__ __forceinline__ float lds(const float* p) { return *p; }
};
// bf16 is carried as raw uint16 bit patterns; widening to fp32 is exact (reading R13).
template <> struct InTraits<uint16_t> {
  static __device__ __forceinline__ float load(const uint16_t* p) {
    return __uint_as_float(static_cast<uint32_t>(__ldg(reinterpret_cast<const unsigned short*>(p))) << 16);
  }
  static __device__ __forceinline__ float lds(const uint16_t* p) { return __uint_as_float(static_cast<uint32_t>(*p) << 16); }
};

// One depth-4 tree walk (a2): node <- 2*node + (v_t > thr[2^t-1+node]); NaN compares false.
__device__ __forceinline__ int tree_walk(const float v[4], const float* thr_t, int C, int c) {
  int node = 0;
#pragma unroll
  for (int t = 0; t < kLevels; ++t) {
    const float th = thr_t[((1 << t) - 1 + node) * C + c];
    node = 2 * node + (v[t] > th ? 1 : 0);
  }
  return node;
}

// Named barriers (bar.sync / bar.arrive) for the producer/consumer ring.
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// 16-bit-lane SWAR widening of 4 uint8 LUT entries: even bytes / odd bytes (one PRMT each).
__device__ __forceinline__ uint32_t even_bytes(uint32_t w) { return __byte_perm(w, 0u, 0x4240); }
__device__ __forceinline__ uint32_t odd_bytes(uint32_t w) { return __byte_perm(w, 0u, 0x4341); }

// acc += x issued as IMAD (x * one + acc) so that the adds run on the FMA pipe and leave the
// ALU pipe to the PRMT widening; `one` is a runtime 1 the compiler cannot fold.
__device__ __forceinline__ void add_fma_pipe(uint32_t& acc, uint32_t x, uint32_t one) {
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc) : "r"(x), "r"(one));
}

// ------------------------------------------------------------------------------ PTX helpers (mbarrier, bulk copy, PDL)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
// Blocking wait for the phase with `parity` to complete: try_wait (the hardware suspends the
// thread for a short, system-defined window per attempt).  After ~2^28 attempts the kernel traps,
// so a broken pipeline protocol surfaces as a launch error instead of a hung GPU.  (A 1 ms
// suspend-time hint compiles to NANOSLEEP.SYNCS, which wakes at any barrier event of the SM: no
// fewer re-checks, and measured no faster; tools/probes/ring_probe.cu gives the ring's costs.)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  for (uint32_t it = 0;; ++it) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    if (ok) return;
    if (it > (1u << 28)) __trap();
  }
}

// Non-blocking test of a phase (warp-uniform when all lanes test the same barrier).
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
// 1-D bulk copy global -> shared (TMA engine, UBLKCP), completion counted on `bar` in bytes.
// dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// L2 eviction-priority policy for cache-hinted copies: 0 = none, 1 = evict_first, 2 = evict_last.
__device__ __forceinline__ uint64_t l2_policy(int kind) {
  uint64_t pol = 0;
  if (kind == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else if (kind == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else if (kind == 3) asm volatile("createpolicy.fractional.L2::evict_first.L2::evict_unchanged.b64 %0, 0.5;" : "=l"(pol));
  else if (kind == 4) asm volatile("createpolicy.fractional.L2::evict_first.L2::evict_unchanged.b64 %0, 0.25;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
// Programmatic dependent launch: wait for the preceding grid's memory to be visible / allow
// the next grid to start its prologue.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Spin (with back-off) until *p >= v, acquire at GPU scope.  Traps after ~10 s so that a broken
// producer/consumer protocol surfaces as a launch error instead of a hung GPU.
__device__ __forceinline__ void spin_until_geq(const uint32_t* p, uint32_t v) {
  uint32_t x;
  for (uint64_t it = 0;; ++it) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(p) : "memory");
    if (x >= v) return;
    __nanosleep(it < 64 ? 32 : 256);
    if (it > (1ull << 25)) __trap();
  }
}

__device__ __forceinline__ uint64_t gtimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float relu_pos0(float y) { return y > 0.0f ? y : 0.0f; }

// One lane of a converged warp (elect.sync): the lane that issues a warp-uniform tcgen05 op.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}
// (float)v for v < 2^23: the bits of 2^23 + v, minus 2^23 (both steps exact).  FMA pipe, not the
// conversion unit (I2F runs on the XU pipe: ncu flagged it saturated in the r01 epilogue).
__device__ __forceinline__ float u2f_exact(uint32_t v) { return __uint_as_float(v | 0x4B000000u) - 8388608.0f; }


__device__ __forceinline__ void st_cs_f4(float* p, float a, float b, float c, float d) {
  __stcs(reinterpret_cast<float4*>(p), make_float4(a, b, c, d));
}

}  // namespace itlumm
