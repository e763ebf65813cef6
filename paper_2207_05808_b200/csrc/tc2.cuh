// tc2.cuh — one-hot x LUT on CTA PAIRS (tcgen05.mma.cta_group::2) for streamed LUTs (large C).
//
// Why: with the LUT too large to stay resident, every 128-row tile of the 1-CTA kernel pulls each
// 32 KB LUT K-block (256 columns) from L2 once; at the int8 MMA rate that is ~117 GB/s per SM of
// L2->SMEM traffic, more than the ring can hide.  A cluster of two CTAs issues
// M=256 MMAs (cta_group::2): each CTA stages its own 128 one-hot rows and HALF of each LUT K-block
// (128 of the 256 columns); the tensor cores of the pair read both halves, so every LUT byte an SM
// fetches now feeds 256 rows.  Each CTA's TMEM holds the s32 accumulators of its own 128 rows.
//
// Roles per CTA (15 warps): 0-3 producers (one row each: codes -> one-hot K-block, K-major
// SWIZZLE_128B; one arrival per CTA per K-block after a named barrier), 4 MMA (leader CTA only:
// waits on the leader's `full` barrier, which both CTAs' producer groups and B forwarders arrive
// on; commits multicast to both CTAs), 5-12 epilogue (TMEM -> fmaf (+ReLU) -> swizzled staging ->
// TMA tensor store; one arrival per warp on the leader's `acce`), 13 codes +
// LUT bulk-copy issuer, 14 forwarder (waits until a LUT half has landed locally, then arrives on
// the leader's `full`).  Results are bit-identical to every other schedule (exact integer MMA,
// same single fmaf).
#pragma once
#include "tc.cuh"

namespace itlumm {

constexpr int kTc2Threads = kTcThreads + 64;      // + LUT forwarder warp + one-hot forwarder warp
constexpr int kTc2FwdWarp = kTcLoaderWarp + 1;    // warp 14
constexpr int kTc2AFwdWarp = kTcLoaderWarp + 2;   // warp 15
constexpr int kTc2Stages = 4;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of `local` in CTA `rank` of this cluster
__device__ __forceinline__ uint32_t mapa_shared(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void umma_i8_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_2sm(uint64_t* bar) {   // arrive on `bar` in both CTAs
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
// Instruction descriptor, kind::i8, M = 256 (pair), N = n.
__host__ __device__ constexpr uint32_t idesc_i8_m256(int n) {
  return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

struct Tc2Smem {
  size_t b, a, stg, codes, bar, tmem, total;
};
// per CTA: a ring of ST one-hot K-blocks (128 rows x 128 B) and a deeper ring of BST half LUT
// K-blocks (128 columns x 128 B): the LUT halves ride the longer L2 -> forwarder -> leader path.
__host__ __device__ inline Tc2Smem tc2_smem_layout(int CS, int ldc, int ST = kTc2Stages, int BST = kTc2Stages) {
  Tc2Smem s{};
  size_t o = 0;
  s.b = o;     o += (size_t)BST * 128 * kKBlock;
  s.a = o;     o += (size_t)ST * kTcRows * kKBlock;
  s.stg = o;   o += (size_t)kTcEpiWarps * kTcStage;
  s.codes = o; o += (size_t)CS * kTcRows * ldc;
  o = (o + 7) & ~(size_t)7;
  s.bar = o;   o += (size_t)(3 * ST + 4 * BST + 4 + 2 * CS) * 8;
  s.tmem = o;  o += 16;
  s.total = o + 1024;
  return s;
}

// NS = 256 columns per slice; g.qt holds [G][KB][256][128 B] (K-major, SW128); scale/offtot padded.
__global__ void __launch_bounds__(kTc2Threads, 1) k_tc2(DevPlan p, TcKArgs g, const __grid_constant__ CUtensorMap out_map) {
  extern __shared__ __align__(1024) uint8_t smem_raw2[];
  uint8_t* smem = smem_raw2 + ((1024u - (smem_u32(smem_raw2) & 1023u)) & 1023u);
  const int C = p.C, KB = g.KB, NS = g.NS, G = g.G, CS = g.CS, ST = g.ST, BST = g.BST;
  const Tc2Smem L = tc2_smem_layout(CS, (int)g.ldc, ST, BST);
  uint8_t* b_s = smem + L.b;
  uint8_t* a_s = smem + L.a;
  uint8_t* codes_s = smem + L.codes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L.bar);   // leader: one-hot of both CTAs (2)
  uint64_t* empty_bar = full_bar + ST;                                // multicast MMA commit (one-hot)
  uint64_t* bready_bar = empty_bar + ST;                              // leader: LUT halves of both CTAs (2)
  uint64_t* bempty_bar = bready_bar + BST;                            // multicast MMA commit (LUT)
  uint64_t* bfull_bar = bempty_bar + BST;                             // local: LUT half landed
  uint64_t* bfwd_bar = bfull_bar + BST;                               // local: forwarder done with stage
  uint64_t* afull_bar = bfwd_bar + BST;                               // local: 128 producers wrote the stage
  uint64_t* accf_bar = afull_bar + ST;                                // multicast MMA commit
  uint64_t* acce_bar = accf_bar + 2;                                  // leader: 2 x 256 epilogue threads
  uint64_t* codes_bar = acce_bar + 2;
  uint64_t* codes_empty = codes_bar + CS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem);

  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1, npair = gridDim.x >> 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* trace = (g.trace && blockIdx.x < 8) ? g.trace + (size_t)blockIdx.x * 4 * kTraceEv : nullptr;
  int tev[4] = {0, 0, 0, 0};
  auto stamp = [&](int role) {                          // 0 producer, 1 MMA, 2 epilogue, 3 loader/fwd
    if (trace && tev[role] < kTraceEv) trace[role * kTraceEv + tev[role]++] = gtimer();
  };
  constexpr int ROWS = 2 * kTcRows;                                  // rows per item (the pair)
  const int64_t ntiles = (g.N + ROWS - 1) / ROWS;
  const int64_t units = ntiles * G;
  auto item = [&](int64_t k, int64_t& tile, int& sl) -> bool {
    const int64_t u = pair + k * npair;
    sl = (int)(u / ntiles);
    tile = u - (int64_t)sl * ntiles;
    return u < units;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(full_bar + s, 2);                 // the one-hot forwarders of the pair
      mbar_init(empty_bar + s, 1);
      mbar_init(afull_bar + s, kTcProducers);
    }
    for (int s = 0; s < BST; ++s) {
      mbar_init(bready_bar + s, 2);               // the 2 forwarders of the pair
      mbar_init(bempty_bar + s, 1);
      mbar_init(bfull_bar + s, 1);
      mbar_init(bfwd_bar + s, 1);
    }
    for (int a = 0; a < 2; ++a) { mbar_init(accf_bar + a, 1); mbar_init(acce_bar + a, 2 * kTcEpiWarps); }
    for (int s = 0; s < CS; ++s) { mbar_init(codes_bar + s, 1); mbar_init(codes_empty + s, kTcProducers); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kTcMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(g.tmem_cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();                                   // peer barriers initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (g.pdl) pdl_wait();
  const uint32_t full_leader = mapa_shared(smem_u32(full_bar), 0);
  const uint32_t bready_leader = mapa_shared(smem_u32(bready_bar), 0);
  const uint32_t acce_leader = mapa_shared(smem_u32(acce_bar), 0);

  if (warp == kTcLoaderWarp) {
    // ======================================================== codes (own 128 rows) + LUT halves
    if (lane == 0) {
      int cs = 0, stage = 0;
      uint32_t cph = 0, phase = 0;
      const uint32_t hbytes = 128u * kKBlock;                        // half LUT K-block
      int64_t tile;
      int sl;
      for (int64_t k = 0; item(k, tile, sl); ++k) {
        mbar_wait(codes_empty + cs, cph ^ 1);
        const int64_t r0 = tile * ROWS + (int64_t)rank * kTcRows;
        const int64_t rows = g.N - r0 < kTcRows ? (g.N - r0 > 0 ? g.N - r0 : 0) : kTcRows;
        mbar_arrive_expect_tx(codes_bar + cs, (uint32_t)(rows * g.ldc));
        if (rows > 0) bulk_g2s(codes_s + (size_t)cs * kTcRows * g.ldc, g.codes + r0 * g.ldc, (uint32_t)(rows * g.ldc), codes_bar + cs);
        if (++cs == CS) { cs = 0; cph ^= 1; }
        const uint8_t* src = g.qt + ((size_t)sl * KB * NS + (size_t)rank * 128) * kKBlock;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(bempty_bar + stage, phase ^ 1);                 // pair's MMAs done with the stage
          mbar_wait(bfwd_bar + stage, phase ^ 1);                   // forwarder saw the previous fill
          mbar_arrive_expect_tx(bfull_bar + stage, hbytes);
          bulk_g2s(b_s + (size_t)stage * hbytes, src + (size_t)kb * NS * kKBlock, hbytes, bfull_bar + stage);
          if (++stage == BST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == kTc2FwdWarp) {
    // ======================================================== forwarder: LUT half landed -> leader
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int64_t tile;
      int sl;
      for (int64_t k = 0; item(k, tile, sl); ++k)
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(bfull_bar + stage, phase);
          mbar_arrive_cluster(bready_leader + stage * 8);
          stamp(3);
          mbar_arrive(bfwd_bar + stage);
          if (++stage == BST) { stage = 0; phase ^= 1; }
        }
    }
  } else if (warp == kTc2AFwdWarp) {
    // ======================================================== one-hot forwarder: stage -> leader
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int64_t tile;
      int sl;
      for (int64_t k = 0; item(k, tile, sl); ++k)
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(afull_bar + stage, phase);
          mbar_arrive_cluster(full_leader + stage * 8);
          if (++stage == ST) { stage = 0; phase ^= 1; }
        }
    }
  } else if (warp < kTcProducerWarps) {
    // ======================================================== producers: one row each
    const int r = threadIdx.x;
    int stage = 0, cs = 0;
    uint32_t phase = 0, cph = 0;
    int64_t tile;
    int sl;
    for (int64_t k = 0; item(k, tile, sl); ++k) {
      mbar_wait(codes_bar + cs, cph);
      const bool valid = tile * ROWS + (int64_t)rank * kTcRows + r < g.N;
      const uint8_t* crow = codes_s + ((size_t)cs * kTcRows + r) * g.ldc;
      for (int kb = 0; kb < KB; ++kb) {
        const uint32_t cw = valid ? *reinterpret_cast<const uint32_t*>(crow + kb * 4) : 0u;
        mbar_wait(empty_bar + stage, phase ^ 1);
        uint8_t* st = a_s + (size_t)stage * kTcRows * kKBlock;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = kb * 8 + j;
          const uint32_t kk = (cw >> (4 * j)) & 15u;
          const uint32_t bit = (valid && c < C) ? (1u << ((kk & 3u) * 8u)) : 0u;
          const uint32_t w = kk >> 2;
          *reinterpret_cast<uint4*>(st + sw128_off(r, j)) =
              make_uint4(w == 0 ? bit : 0u, w == 1 ? bit : 0u, w == 2 ? bit : 0u, w == 3 ? bit : 0u);
        }
        // producers release their one-hot stores locally (CTA scope); the one-hot forwarder warp
        // turns each completed stage into one cluster-scope arrival on the leader, off the
        // producers' critical path
        fence_proxy_async_smem();
        mbar_arrive(afull_bar + stage);
        if (r == 0) stamp(0);
        if (++stage == ST) { stage = 0; phase ^= 1; }
      }
      mbar_arrive(codes_empty + cs);
      if (++cs == CS) { cs = 0; cph ^= 1; }
    }
  } else if (warp == kTcMmaWarp) {
    // ======================================================== MMA: leader CTA issues for the pair
    if (rank == 0) {
      const uint32_t idesc = idesc_i8_m256(NS);
      int stage = 0, acc = 0, bstage = 0;
      uint32_t phase = 0, acc_phase = 0, bphase = 0;
      int64_t tile;
      int sl;
      for (int64_t k = 0; item(k, tile, sl); ++k) {
        mbar_wait(acce_bar + acc, acc_phase ^ 1);                  // both epilogues drained it
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * NS);
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(full_bar + stage, phase);
          mbar_wait(bready_bar + bstage, bphase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(a_s + (size_t)stage * kTcRows * kKBlock);
            const uint32_t b_addr = smem_u32(b_s + (size_t)bstage * 128 * kKBlock);
#pragma unroll
            for (int ks = 0; ks < kKBlock / 32; ++ks)
              umma_i8_2sm(d, umma_desc_sw128(a_addr + ks * 32), umma_desc_sw128(b_addr + ks * 32), idesc,
                          (kb | ks) != 0);
            umma_commit_2sm(empty_bar + stage);
            umma_commit_2sm(bempty_bar + bstage);
            if (kb == KB - 1) umma_commit_2sm(accf_bar + acc);
            stamp(1);
          }
          __syncwarp();
          if (++stage == ST) { stage = 0; phase ^= 1; }
          if (++bstage == BST) { bstage = 0; bphase ^= 1; }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ======================================================== epilogue (own 128 rows, 256 columns)
    const int e = warp - kTcEpiWarp0;
    const int q = warp & 3;
    const int h = e >> 2;
    uint8_t* stg = smem + L.stg + (size_t)e * kTcStage;
    int acc = 0;
    uint32_t acc_phase = 0;
    bool pending = false;
    int64_t tile;
    int sl;
    for (int64_t k = 0; item(k, tile, sl); ++k) {
      mbar_wait(accf_bar + acc, acc_phase);
      tc_fence_after();
      if (e == 0 && lane == 0) stamp(2);
      const int m0 = sl * NS;
      const int row0 = (int)(tile * ROWS) + (int)rank * kTcRows + q * 32;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * NS);
      for (int j0 = h * 32; j0 < NS; j0 += 64) {
        uint32_t v[32];
        tmem_ld16(tbase + j0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
        tmem_ld16(tbase + j0 + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
        tmem_wait_ld();
        float y[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 s4 = __ldg(reinterpret_cast<const float4*>(p.scale + m0 + j0 + 4 * c));
          const float4 o4 = __ldg(reinterpret_cast<const float4*>(p.offtot + m0 + j0 + 4 * c));
          y[4 * c + 0] = fmaf(s4.x, __uint2float_rn(v[4 * c + 0]), o4.x);   // a4, one rounding (R8)
          y[4 * c + 1] = fmaf(s4.y, __uint2float_rn(v[4 * c + 1]), o4.y);
          y[4 * c + 2] = fmaf(s4.z, __uint2float_rn(v[4 * c + 2]), o4.z);
          y[4 * c + 3] = fmaf(s4.w, __uint2float_rn(v[4 * c + 3]), o4.w);
        }
        if (g.relu) {
#pragma unroll
          for (int j = 0; j < 32; ++j) y[j] = relu_pos0(y[j]);
        }
        if (pending) {
          if (lane == 0) bulk_wait_read0();
          __syncwarp();
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<float4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) =
              make_float4(y[4 * c], y[4 * c + 1], y[4 * c + 2], y[4 * c + 3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&out_map, stg, m0 + j0, row0);
          bulk_commit();
        }
        pending = true;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acce_leader + acc * 8);
      if (e == 0 && lane == 0) stamp(2);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) bulk_wait0();
  }

  tc_fence_before();
  cluster_sync_all();                                   // the pair is done with TMEM and barriers
  if (warp == kTcMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(g.tmem_cols) : "memory");
  }
}

}  // namespace itlumm

namespace itlumm {

// Launch k_tc2 for a streamed-LUT plan when it applies (codes path, TMA-storable output, no int32
// acc output, 256-column slices, 16-byte codes rows).  Returns false (nothing launched) otherwise.
// OFF by default: measured slower than the 1-CTA streamed kernel (cfg3 C=64 / C=128 / cfg5:
// 83 / 140 / 5090 us vs 61 / 101 / 3560 us).  With the one-hot and LUT rings decoupled and their
// cluster-scope arrivals moved to forwarder warps, the K-block cadence settles at ~650 ns for any
// ring depth from 3 to 7 (profiles/r01/tc2_stage_sweep.txt), i.e. a throughput limit of the pair
// MMA path rather than latency.  Parity-exact; opt in with ITLUMM_TC2=1 (developer knob, not ABI).
inline bool tc2_applicable(const TcPlan& t, const TcArgs& a) {
  static const bool on = getenv("ITLUMM_TC2") && atoi(getenv("ITLUMM_TC2")) != 0;
  return on && t.stream_b && t.NS == 256 && t.tmem_cols == 512 && !a.acc && a.out && a.ldc % 16 == 0 &&
         (reinterpret_cast<uintptr_t>(a.codes) & 15) == 0 && a.N > 0;
}

inline itlumm_status tc2_launch(const TcPlan& t, const DevPlan& dp, const TcArgs& a, cudaStream_t s, int num_sms,
                                bool pdl, bool* launched) {
  *launched = false;
  if (!tc2_applicable(t, a)) return ITLUMM_OK;
  alignas(64) CUtensorMap out_map;
  memset(&out_map, 0, sizeof out_map);
  if (!make_out_map(&out_map, a.out, a.N, t.M, a.ldo)) return ITLUMM_OK;
  // one-hot and LUT-half rings of similar depth (the cross-CTA round trip is long on both), 2 codes
  // stages (1 if short of room).  Developer override (not ABI): ITLUMM_TC2_ST.
  static const int st_env = getenv("ITLUMM_TC2_ST") ? atoi(getenv("ITLUMM_TC2_ST")) : 0;
  int ST = (st_env >= 2 && st_env <= 8) ? st_env : 5;
  int CS = 2, BST = 0;
  if (tc2_smem_layout(CS, (int)a.ldc, ST, 4).total > kSmemMax) CS = 1;
  while (BST < 8 && tc2_smem_layout(CS, (int)a.ldc, ST, BST + 1).total <= kSmemMax) ++BST;
  while (BST < 3 && ST > 2) {
    --ST;
    while (BST < 8 && tc2_smem_layout(CS, (int)a.ldc, ST, BST + 1).total <= kSmemMax) ++BST;
  }
  if (BST < 2 || (int64_t)kTcRows * a.ldc >= (1 << 20)) return ITLUMM_OK;
  const size_t smem = tc2_smem_layout(CS, (int)a.ldc, ST, BST).total;
  static bool attr_done = false;
  if (!attr_done) {
    if (cudaFuncSetAttribute((const void*)k_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax) != cudaSuccess)
      return ITLUMM_OK;
    attr_done = true;
  }
  TcKArgs k{};
  k.codes = a.codes; k.ldc = a.ldc; k.N = a.N; k.out = a.out; k.ldo = a.ldo; k.relu = a.relu;
  k.qt = t.qt; k.KB = t.KB; k.NS = t.NS; k.G = t.G; k.tmem_cols = t.tmem_cols;
  k.CS = CS; k.pdl = pdl ? 1 : 0; k.tma_store = 1; k.ST = ST; k.BST = BST; k.stream_b = 1;
  k.trace = t.trace;
  const int64_t units = ((a.N + 255) / 256) * t.G;
  int64_t pairs = num_sms / 2;
  if (pairs > units) pairs = units;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(2 * pairs));
  cfg.blockDim = dim3(kTc2Threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_tc2, dp, k, out_map);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) { g_tc_msg = cudaGetErrorString(e); return ITLUMM_ECUDA; }
  *launched = true;
  return ITLUMM_OK;
}

}  // namespace itlumm
