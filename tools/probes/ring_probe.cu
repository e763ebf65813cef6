// ring_probe.cu — developer probe: the cost of the producer -> MMA -> producer ring protocol alone.
//
// One CTA per SM (or a CTA pair), no data: P producer warps loop over the stages: wait `empty[s]`,
// (optionally) store 16 B per thread into a stage buffer + fence.proxy.async, then arrive on
// `full[s]`: per THREAD (128/256 arrivals), per WARP (lane 0 after __syncwarp), or per CTA (named
// barrier over the producers, then one thread).  One MMA warp waits `full[s]` and answers with
// tcgen05.commit to `empty[s]` (no MMA: the commit arrives once prior tcgen05 ops are done, here
// none), or with tcgen05.mma (4 x N=256 i8 from the stage) then the commit.  Reports cycles per stage.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  for (uint32_t it = 0;; ++it) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
    if (ok) return;
    if (it > (1u << 28)) __trap();
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ uint64_t mdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// mode: 0 per-thread arrive, 1 per-warp arrive, 2 per-CTA (named barrier + 1 arrive)
template <int MODE, bool STORE, bool MMA, bool LOADB, int EPI>
__global__ void k_ring(int P, int ST, int stages, unsigned long long* out, const uint8_t* lut, float* gout,
                       const __grid_constant__ CUtensorMap omap_v, const uint8_t* ga) {
  const CUtensorMap* omap = &omap_v;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
  uint8_t* ring = sm;                                    // ST x 48 KB (A 16 KB + B 32 KB)
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)ST * 49152);
  uint64_t* empty = full + ST;
  uint64_t* accf = empty + ST;          // [2] MMA -> epilogue
  uint64_t* acce = accf + 2;            // [2] epilogue -> MMA
  uint32_t* slot = reinterpret_cast<uint32_t*>(acce + 2);
  constexpr int KB = 32;                // stages per item (accumulator), as cfg5 (C = 256)
  const int loader_warp = P + 1, epi0 = P + 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nprod = 32 * P;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(full + s, MODE == 8 ? 1 : (MODE == 0 || MODE >= 3 ? nprod : MODE == 1 ? P : 1) + (LOADB ? 1 : 0));
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) { mbar_init(accf + a, 1); mbar_init(acce + a, 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == P) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = *slot;
  unsigned long long t0 = clock64();
  if (warp < P && MODE != 8) {
    int st = 0;
    uint32_t ph = 0;
    for (int i = 0; i < stages; ++i) {
      mbar_wait(empty + st, ph ^ 1);
      if (MODE == 6 || MODE == 7) {
        // A operand in TMEM: warp q writes the one-hot rows 32q..32q+31 (its TMEM lane quadrant),
        // 32 columns (128 B) per stage, one tcgen05.st.32x32b.x32 per warp
        const int r = threadIdx.x & 127;
        const uint32_t cw = *reinterpret_cast<const uint32_t*>(ring + 16384 + r * 132 + (i & 31) * 4);
        uint32_t a[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t k = (cw >> (4 * j)) & 15u;
          const uint32_t bit = 1u << ((k & 3u) * 8u);
          const uint32_t w = k >> 2;
          a[4 * j + 0] = w == 0 ? bit : 0u; a[4 * j + 1] = w == 1 ? bit : 0u;
          a[4 * j + 2] = w == 2 ? bit : 0u; a[4 * j + 3] = w == 3 ? bit : 0u;
        }
        const uint32_t taddr = tm + ((uint32_t)((warp & 3) * 32) << 16) + (MODE == 7 ? 448u : 384u) + 32u * st;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                     "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
                     "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]),
                     "r"(a[8]), "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]), "r"(a[14]), "r"(a[15]),
                     "r"(a[16]), "r"(a[17]), "r"(a[18]), "r"(a[19]), "r"(a[20]), "r"(a[21]), "r"(a[22]), "r"(a[23]),
                     "r"(a[24]), "r"(a[25]), "r"(a[26]), "r"(a[27]), "r"(a[28]), "r"(a[29]), "r"(a[30]), "r"(a[31]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        mbar_arrive(full + st);
        if (++st == ST) { st = 0; ph ^= 1; }
        continue;
      }
      if (MODE == 4 || MODE == 5) {
        // MODE 4: 5 STS.128 per row (the 2:4-sparse volume: 64 B values + 16 B metadata);
        // MODE 5: two threads per row (8 producer warps), 4 STS.128 each
        const int r = threadIdx.x & 127, half = threadIdx.x >> 7;
        const uint32_t cw = *reinterpret_cast<const uint32_t*>(ring + 16384 + r * 132 + (i & 31) * 4);
        uint8_t* stg = ring + (size_t)st * 49152;
        const int nj = MODE == 4 ? 5 : 4;
#pragma unroll
        for (int jj = 0; jj < nj; ++jj) {
          const int j = MODE == 4 ? jj : 4 * half + jj;
          const uint32_t k = (cw >> (4 * (j & 7))) & 15u;
          const uint32_t bit = 1u << ((k & 3u) * 8u);
          const uint32_t w = k >> 2;
          const uint32_t off = (r >> 3) * 1024u + (r & 7u) * 128u + (((j & 7) ^ (r & 7u)) << 4);
          *reinterpret_cast<uint4*>(stg + off) =
              make_uint4(w == 0 ? bit : 0u, w == 1 ? bit : 0u, w == 2 ? bit : 0u, w == 3 ? bit : 0u);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(full + st);
        if (++st == ST) { st = 0; ph ^= 1; }
        continue;
      }
      if (MODE == 3) {
        // as k_tc's producers: the row's 4 code bytes of this K-block from a codes tile in smem
        // (the codes live in the B region of stage 0 here: timing only), 8 dense one-hot chunks in
        // the SWIZZLE_128B K-major layout
        const int r = threadIdx.x & 127;
        const uint32_t cw = *reinterpret_cast<const uint32_t*>(ring + 16384 + r * 132 + (i & 31) * 4);
        uint8_t* stg = ring + (size_t)st * 49152;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t k = (cw >> (4 * j)) & 15u;
          const uint32_t bit = 1u << ((k & 3u) * 8u);
          const uint32_t w = k >> 2;
          const uint32_t off = (r >> 3) * 1024u + (r & 7u) * 128u + ((j ^ (r & 7u)) << 4);
          *reinterpret_cast<uint4*>(stg + off) =
              make_uint4(w == 0 ? bit : 0u, w == 1 ? bit : 0u, w == 2 ? bit : 0u, w == 3 ? bit : 0u);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(full + st);
        if (++st == ST) { st = 0; ph ^= 1; }
        continue;
      }
      if (STORE) {
        uint8_t* a = ring + (size_t)st * 49152 + threadIdx.x * 16;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(su32(a + (j * nprod * 16) % 16384)), "r"(i) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      if (MODE == 0) {
        mbar_arrive(full + st);
      } else if (MODE == 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive(full + st);
      } else {
        asm volatile("bar.sync 1, %0;" ::"r"(nprod) : "memory");
        if (threadIdx.x == 0) mbar_arrive(full + st);
      }
      if (++st == ST) { st = 0; ph ^= 1; }
    }
  } else if (warp == P) {
    int st = 0, acc = 0;
    uint32_t ph = 0, aph = 0;
    const uint32_t idesc = (2u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    for (int i = 0; i < stages; ++i) {
      const int kb = i % KB;
      if (EPI && kb == 0) mbar_wait(acce + acc, aph ^ 1);
      mbar_wait(full + st, ph);
      uint32_t e;
      asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(e));
      if (e) {
        if (MMA && (MODE == 6 || MODE == 7)) {
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t bd = mdesc(su32(ring + (size_t)st * 49152 + 16384));
          constexpr uint32_t NN = MODE == 7 ? 224u : 192u;
          const uint32_t id192 = (2u << 4) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + NN * acc),
                         "r"(tm + 2u * NN + 32u * st + 8u * k), "l"(bd + 2 * k), "r"(id192), "r"(kb | k) : "memory");
        } else if (MMA) {
          const uint64_t ad = mdesc(su32(ring + (size_t)st * 49152)), bd = mdesc(su32(ring + (size_t)st * 49152 + 16384));
#pragma unroll
          for (int k = 0; k < 4; ++k)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm + 256u * acc), "l"(ad + 2 * k), "l"(bd + 2 * k),
                         "r"(idesc), "r"(kb | k) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(empty + st)) : "memory");
        if (EPI && kb == KB - 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(accf + acc)) : "memory");
      }
      __syncwarp();
      if (++st == ST) { st = 0; ph ^= 1; }
      if (EPI && kb == KB - 1 && ++acc == 2) { acc = 0; aph ^= 1; }
    }
    for (int s = 0; s < ST; ++s) {
      const int idx = stages - ST + s;
      if (idx < 0) continue;
      mbar_wait(empty + (idx % ST), (uint32_t)((idx / ST) & 1));
    }
    if (blockIdx.x == 0 && lane == 0) out[0] = clock64() - t0;
  } else if (warp == loader_warp) {
    if (LOADB && lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int i = 0; i < stages; ++i) {
        mbar_wait(empty + st, ph ^ 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + st)), "r"(MODE == 8 ? 49152 : 32768) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(ring + (size_t)st * 49152 + 16384)), "l"(lut + (size_t)(i % 512) * 32768), "r"(32768),
                     "r"(su32(full + st)) : "memory");
        if (MODE == 8)   // A from a 1 GB one-hot matrix in HBM: this CTA's rows, K-block i
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(ring + (size_t)st * 49152)), "l"(ga + ((size_t)blockIdx.x * 4096 + (size_t)(i % 4096)) * 16384 % (1ull << 30)),
                       "r"(16384), "r"(su32(full + st)) : "memory");
        if (++st == ST) { st = 0; ph ^= 1; }
      }
    }
  } else if (EPI && warp >= epi0 && warp < epi0 + 8) {
    const int e = warp - epi0, q = warp & 3, h = e >> 2;
    int acc = 0;
    uint32_t aph = 0;
    const int items = stages / KB;
    for (int it = 0; it < items; ++it) {
      mbar_wait(accf + acc, aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      constexpr uint32_t NCOL = MODE == 6 ? 192u : MODE == 7 ? 224u : 256u;
      const uint32_t tb = tm + ((uint32_t)(q * 32) << 16) + NCOL * acc;
      for (int j0 = h * 32; j0 < (int)NCOL; j0 += 64) {
        uint32_t v[16];
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          if (EPI == 3) {
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = c + it;
          } else
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                       : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                         "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                       : "r"(tb + j0 + 16 * half));
          if (EPI != 3) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (EPI == 2) { if (v[0] == 0xFFFFFFFFu && v[15] == 7u) gout[lane] = 1.f; continue; }
          if (EPI == 5 || EPI == 6) {
            // EPI 5: 32 lanes x 16 B contiguous (512 B per instruction); EPI 6: 8 lanes per 128 B row
            // segment, 4 rows per instruction
            const size_t rowbase = (size_t)(blockIdx.x * 128 + q * 32) * 256 + j0 + 16 * half;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              size_t off = EPI == 5 ? ((rowbase + (size_t)(c * 8 + lane / 4) * 256) + (lane & 3) * 4)
                                    : ((rowbase + (size_t)(c * 8 + lane / 8 * 2) * 256) + (lane & 7) * 4);
              float* o = gout + off % ((1u << 24) - 4);
              reinterpret_cast<float4*>(o)[0] = make_float4(__uint_as_float(v[4 * c]), __uint_as_float(v[4 * c + 1]),
                                                            __uint_as_float(v[4 * c + 2]), __uint_as_float(v[4 * c + 3]));
            }
            continue;
          }
          if (EPI == 7) {
            // as k_tc's epilogue: 32 rows x 32 fp32 box, 128B-swizzled staging, 2-D tensor store
            uint8_t* stg = ring + 8192 + (warp & 7) * 4096 - 8192 * 0;
            if (half == 0) {
              // stage the first 16 columns now, the second 16 on the next half (one 32x32 box per j0)
            }
#pragma unroll
            for (int c = 0; c < 4; ++c)
              *reinterpret_cast<uint4*>(stg + lane * 128 + (((c + 4 * half) ^ (lane & 7)) << 4)) =
                  make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
            if (half == 1) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              __syncwarp();
              if (lane == 0) {
                const int x = j0, y = (blockIdx.x * 128 + q * 32) % 16384;
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];"
                             ::"l"(reinterpret_cast<uint64_t>(omap)), "r"(su32(stg)), "r"(x), "r"(y) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              }
              __syncwarp();
            }
            continue;
          }
          if (EPI == 4) {
            // staging in shared memory (the A region of stage 0 is reused: timing only) + 1-D bulk store
            uint8_t* stg = ring + 8192 + (warp & 7) * 1024;
#pragma unroll
            for (int c = 0; c < 4; ++c)
              *reinterpret_cast<uint4*>(stg + lane * 16 + c * 512 - (c * 512 + lane * 16 >= 1024 ? 1024 : 0)) =
                  make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              float* o = gout + ((size_t)(blockIdx.x * 128 + q * 32) * 256 + j0 * 32 + half * 256) % ((1u << 24) - 256);
              asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(o), "r"(su32(stg)), "r"(1024) : "memory");
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
              asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncwarp();
            continue;
          }
          float* o = gout + ((size_t)(blockIdx.x * 128 + q * 32 + lane) * 256 + j0 + 16 * half) % (1u << 24);
#pragma unroll
          for (int c = 0; c < 4; ++c)
            reinterpret_cast<float4*>(o)[c] = make_float4(__uint_as_float(v[4 * c]) * 1.5f, __uint_as_float(v[4 * c + 1]),
                                                          __uint_as_float(v[4 * c + 2]), __uint_as_float(v[4 * c + 3]));
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(acce + acc);
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == P) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

static CUtensorMap g_omap;
static const uint8_t* g_a;
template <int MODE, bool STORE, bool MMA, bool LOADB, int EPI>
static void run(int sms, int P, int ST, unsigned long long* d, const uint8_t* lut, float* gout) {
  const int stages = 32 * 640;
  const size_t smem = (size_t)ST * 49152 + 1024 + 256;
  auto k = k_ring<MODE, STORE, MMA, LOADB, EPI>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int threads = 32 * (P + 2 + 8);
  k<<<sms, threads, smem>>>(P, ST, 32 * 8, d, lut, gout, g_omap, g_a);
  k<<<sms, threads, smem>>>(P, ST, stages, d, lut, gout, g_omap, g_a);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); exit(1); }
  unsigned long long cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  printf("{\"mode\": \"%s\", \"store\": %d, \"mma\": %d, \"loadb\": %d, \"epi\": %d, \"producer_warps\": %d, \"stages_in_ring\": %d, \"cycles_per_stage\": %.1f}\n",
         MODE == 0 ? "per-thread" : MODE == 1 ? "per-warp" : MODE == 2 ? "per-cta" : MODE == 3 ? "k_tc-producer" : MODE == 4 ? "5-sts" : MODE == 5 ? "2-threads-per-row" : MODE == 6 ? "A-in-TMEM N=192" : MODE == 7 ? "A-in-TMEM N=224" : "A by TMA from HBM", (int)STORE, (int)MMA, (int)LOADB, (int)EPI, P, ST, (double)cyc / stages);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, 8);
  uint8_t* lut;
  cudaMalloc(&lut, 16 << 20);
  cudaMemset(lut, 1, 16 << 20);
  float* gout;
  cudaMalloc(&gout, 64 << 20);
  {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    const cuuint64_t dims[2] = {256, 16384};
    const cuuint64_t strides[1] = {256 * 4};
    const cuuint32_t box[2] = {32, 32}, estr[2] = {1, 1};
    CUresult r = enc(&g_omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, gout, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("tensor map failed\n"); return 1; }
  }
  {
    uint8_t* a;
    cudaMalloc(&a, 1ull << 30);
    cudaMemset(a, 1, 1ull << 30);
    g_a = a;
  }
  run<3, true, true, true, 7>(sms, 4, 4, d, lut, gout);
  run<8, true, true, true, 7>(sms, 4, 4, d, lut, gout);
  run<8, true, true, true, 0>(sms, 4, 4, d, lut, gout);
  return 0;
}
