// tcp.cuh — one-hot x LUT on CTA PAIRS (tcgen05.mma.cta_group::2), streamed LUT.
//
// What it computes: a3' + a4 for the shapes whose LUT is too large to stay in shared memory (large C:
// cfg3, cfg4 hidden layers with C >= 64, cfg5's 16 MB LUT).  acc = G.Q exactly, G the one-hot
// encoding of the codes ("the concatenation of C one-hot 16-dimensional vectors"), Q the uint8
// LUT as 16C x M; then y = fmaf(scale, (float)acc, offtot) (+ReLU) (reading R8, R9).
//
// Why this shape (measured, profiles/r02/smem_contention.jsonl, profiles/r02/sp2_probe.txt):
//   * the tcgen05 i8 MMA rate is NOT slowed by other shared-memory traffic (STS at 85 B/clk, TMA at
//     66 B/clk alongside: 128 cycles per N=256 MMA either way), so the one-hot writes are not a
//     bandwidth problem — what bounded the 1-CTA kernel was its ring round trip and producer work;
//   * the 2:4-sparse one-hot (a 1-of-16 vector is always 2:4 sparse) on a CTA pair runs K=64 per
//     128 cycles at N=256: twice the dense K per cycle, where the 1-CTA sparse MMA gains only 1.6x;
//   * a CTA pair stages HALF of every LUT K-block per SM (each LUT byte fetched from L2 feeds 256
//     rows), which halves the L2 -> shared-memory stream that the streamed LUT needs.
//
// Per pair item = (256 rows, one NS-column slice), CTA r of the pair owns rows [128r, 128r+128).
// The ring moves in SLOTS of SS K-blocks (8 codebooks each; SS = 2 by default): one barrier round
// trip, one producer proxy fence + arrive and one MMA commit per slot.  The bare handshakes cost as
// much per slot as per K-block, so two K-blocks per slot halved them (cfg5 accumulate 3.68 -> 2.93
// ms on one box).  Roles (warp -> role: tcp_role):
//   producers (8 warps, SMSPs 1-3)  two threads per row; per K-block of the slot the row's one-hot
//               (dense: 16 B per codebook, K-major SWIZZLE_128B; 2:4-sparse: 8 B per codebook,
//               SWIZZLE_64B, + 16 B of metadata for tcgen05.cp); fence.proxy.async; one arrive per
//               warp and slot on the LEADER's full[st].
//   MMA issuer (warp 0, leader CTA only)  per K-block 4 tcgen05.mma.cta_group::2.kind::i8 (M=256,
//               N=NS, K=32) or, 2:4-sparse, one tcgen05.cp.cta_group::2 of both CTAs' metadata and 2
//               tcgen05.mma.sp (K=64); commits multicast to both CTAs (slot free; accumulator ready).
//   epilogue (8 warps, two per TMEM lane quadrant)  each CTA its own 128 rows: tcgen05.ld -> fmaf
//               (+ReLU) -> 128B-swizzled staging -> TMA tensor store of 32x32 boxes; per-warp
//               arrive on the leader's acce.
//   LUT loader (warp 4)  its half of each LUT K-block (TMA tensor load .cta_group::2: the bytes
//               complete on the LEADER's full[st]).
//   codes loader (warp 16)  the CTA's 128-row codes tile per item (bulk copy), up to CS items ahead;
//               with CS = 0 (developer option) the producers load their codes from global memory.
// Results are bit-identical to every other schedule (exact integer MMA, the same single fmaf).
#pragma once
#include "tc.cuh"

namespace itlumm {

constexpr int kTcpDense = 0, kTcpSparse = 1;   // k_tcp MODE

// Roles: 8 producer warps (two threads per row, four codebooks each), 1 MMA warp, 8 epilogue warps
// (two per TMEM lane quadrant), 1 loader warp.  Two threads per row: one producer warp per SM
// sub-partition could not issue a stage's one-hot in time (tcp_trace: 416 ns per stage against
// ~230 ns of sparse MMA; ncu: ALU pipe 47% busy).
// Warp w runs on SM sub-partition (SMSP) w % 4 and may only read TMEM lanes 32 (w % 4) .. +31.
// SMSP 0 hosts the MMA issuer and the loader (and the two quadrant-0 epilogue warps), no producer:
// producer warps sharing the issuer's SMSP ran ~3000 cycles behind the other producers every stage
// (tcp_trace, profiles/r02): the issuer's tcgen05 ops take ~40 cycles of its SMSP each.
constexpr int kTcpSsMax = 3;           // K-blocks per ring slot at most
constexpr int kTcpProdWarps = 8;
constexpr int kTcpEpiWarps = 8;
constexpr int kTcpMmaWarp = 0;
constexpr int kTcpLoaderWarp = 4;
constexpr int kTcpWarps = 19;
constexpr int kTcpThreads = 32 * kTcpWarps;                    // 608
// role of warp w: 0..7 producer index, 8..15 epilogue index (quadrant = w % 4; index 8 + 2q, 9 + 2q),
// 16 MMA, 17 loader, 18 idle (warp 16: SMSP 0's fifth slot, launched only so that SMSP 2 gets its
// third producer, warp 18)
__host__ __device__ constexpr int tcp_role(int w) {
  return w == 0 ? 16 : w == 4 ? 17 : w == 16 ? 18 :
         w == 1 ? 0 : w == 2 ? 1 : w == 3 ? 2 : w == 5 ? 3 : w == 6 ? 4 : w == 7 ? 5 : w == 9 ? 6 : w == 10 ? 7 :
         w == 8 ? 8 : w == 12 ? 9 : w == 13 ? 10 : w == 17 ? 11 : w == 14 ? 12 : w == 18 ? 13 : w == 11 ? 14 : 15;
}
constexpr int kTcpSpNsMax = 224;                 // 2 x NS accumulators + 4 metadata columns per stage <= 512

// shl.b32 clamps shift amounts >= 32 to 32 (result 0); a "negative" amount wraps to a large one.
__device__ __forceinline__ uint32_t shl_clamp(uint32_t x, uint32_t sh) {
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(sh));
  return r;
}
// One codebook's one-hot for code k (k >= 16: none), branch-free.
//   dense (16 B, byte k = 1): word w = 1 << (8k - 32w), clamped to 0 outside [0, 32).
//   2:4 sparse (8 B + 16-bit metadata): the group g = k >> 2 stores the pair of logical positions
//   (e, 3) with values (1, 0) for e = k & 3 < 3, or (0, 3) with values (0, 1) for e = 3 (the byte
//   at 2g + [e == 3] is 1); metadata nibble g = idx0 | idx1 << 2 = 0xC | (e == 3 ? 0 : e), the other
//   nibbles 0 (their values are 0).  The same encoding as put_onehot<true> (tc.cuh).
__device__ __forceinline__ void onehot_dense16(uint32_t k, uint32_t (&w)[4]) {
  const uint32_t sh = k << 3;
  w[0] = shl_clamp(1u, sh);
  w[1] = shl_clamp(1u, sh - 32u);
  w[2] = shl_clamp(1u, sh - 64u);
  w[3] = shl_clamp(1u, sh - 96u);
}
__device__ __forceinline__ void onehot_sparse8(uint32_t k, uint32_t& lo, uint32_t& hi, uint32_t& m16) {
  const uint32_t t = k & (k >> 1) & 1u;                              // e == 3
  const uint32_t sh = ((k & 12u) << 2) | (t << 3) | ((k & 16u) << 2);   // 8 * byte position; 64 if k >= 16
  uint64_t v;
  asm("shl.b64 %0, %1, %2;" : "=l"(v) : "l"(1ull), "r"(sh));          // clamped: 0 for sh >= 64
  lo = (uint32_t)v;
  hi = (uint32_t)(v >> 32);
  m16 = (((k & 3u) ^ (t * 3u)) | 12u) << (k & 12u);
  if (k >= 16u) m16 = 0u;
}

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
// Arrive on an mbarrier of either CTA of the pair.  No .release.cluster: that form compiles to
// MEMBAR.ALL.GPU + ERRBAR + CGAERRBAR before the arrive (ncu: the producers' and epilogue's
// arrivals became the kernel's top stall).  What must be ordered is ordered locally first: the
// producers' one-hot stores by fence.proxy.async (the SM that reads them through the async proxy
// is their own), the epilogue's TMEM reads by tcgen05.wait::ld + tcgen05.fence::before_thread_sync.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void umma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_sp_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t tmem_e,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "tcgen05.mma.sp.cta_group::2.kind::i8 [%0], %1, %2, [%3], %4, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(tmem_e), "r"(idesc | 4u), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_cp_pair_128x128b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::2.128x128b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {   // arrive on `bar` in both CTAs
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
// 2-D tensor load whose transaction bytes complete on an mbarrier of either CTA of the pair
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int x, int y, uint32_t mbar_cluster) {
  asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(mbar_cluster) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_cluster(uint32_t cluster_addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_addr), "r"(bytes)
               : "memory");
}
// Instruction descriptor, kind::i8, M = 256 (pair), N = n.
__host__ __device__ constexpr uint32_t idesc_i8_m256(int n) {
  return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

// Per-CTA shared memory: ST ring slots of SS stages [A | metadata | B half], CS codes tiles (0: the
// codes come straight from global memory), epilogue staging.
struct TcpSmem {
  size_t a_bytes, e_bytes, b_bytes, stage, ring, codes, stg, bar, tmem, trc, total;
};
constexpr int kTcpTrcSlots = 24, kTcpTrcWin = 64, kTcpTrcFirst = 96;   // developer timeline window
__host__ __device__ inline TcpSmem tcp_smem_layout(int mode, int NS, int ST, int CS, int ldc, bool trace = false, int SS = 1) {
  TcpSmem s{};
  const bool sp = mode == kTcpSparse;
  s.a_bytes = sp ? (size_t)kSpA : (size_t)kTcRows * kKBlock;          // 8 KB compressed / 16 KB dense
  s.e_bytes = sp ? (size_t)kTcRows * 16 : 0;                         // metadata rows (tcgen05.cp source)
  s.b_bytes = (size_t)(NS / 2) * kKBlock;                            // half a LUT K-block
  s.stage = (s.a_bytes + s.e_bytes + s.b_bytes + 1023) & ~(size_t)1023;
  s.ring = 0;
  s.codes = s.ring + (size_t)ST * SS * s.stage;   // ST ring slots of SS sub-stages (one K-block each)
  s.stg = s.codes + (((size_t)CS * kTcRows * ldc + 1023) & ~(size_t)1023);
  s.bar = s.stg + (size_t)kTcEpiWarps * kTcStage;
  s.tmem = s.bar + (size_t)(2 * ST + 4 + 2 * CS) * 8;
  s.trc = s.tmem + 16;
  s.total = s.trc + (trace ? (size_t)kTcpTrcSlots * kTcpTrcWin * 8 : 0) + 1024;   // + slack for 1024-byte alignment
  return s;
}

struct TcpKArgs {
  const uint8_t* codes; int64_t ldc;   // row-major nibble-packed codes, ldc % 16 == 0
  int64_t N;
  int32_t* acc; int64_t ldacc;         // optional raw int32 accumulators (then per-thread stores)
  float* out; int64_t ldo;
  int relu;
  int KB, NS, G, ST, CS;                // KB: 8-codebook K-blocks per item; ST ring slots
  int SS;                              // K-blocks (sub-stages) per ring slot: one barrier round trip each
  int tmem_cols;
  int pdl;
  uint64_t* trace;                     // developer timeline (ITLUMM_TC_TRACE=1): [4 CTAs][4 roles][kTraceEv]
  int cload;                           // codes tiles loaded by their own warp (16) instead of the LUT loader
  int out_hint;                        // L2 policy of the output tensor stores (l2_policy kind; chosen in tcp_launch)
  int dbg;                             // developer removal switches (ITLUMM_TCP_DBG; results then wrong):
                                       // 1 producers skip the one-hot stores, 2 no MMAs (commits only),
                                       // 4 no LUT loads, 8 producers skip fence.proxy.async,
                                       // 16 epilogue skips the output stores, 32 no epilogue work,
                                       // 1024 dense one-hot as zero chunk + one byte store,
                                       // 4096 one ring stage per MMA issue pass
};

template <int MODE>
__global__ void __launch_bounds__(kTcpThreads, 1)
k_tcp(DevPlan p, TcpKArgs g, const __grid_constant__ CUtensorMap out_map, const __grid_constant__ CUtensorMap qt_map) {
  constexpr bool SP = MODE == kTcpSparse;
  extern __shared__ __align__(1024) uint8_t smem_tcp[];
  uint8_t* smem = smem_tcp + ((1024u - (smem_u32(smem_tcp) & 1023u)) & 1023u);
  const int C = p.C, KB = g.KB, NS = g.NS, G = g.G, ST = g.ST, CS = g.CS, SS = g.SS;
  const int KBS = (KB + SS - 1) / SS;      // ring slots per item (the last may hold fewer K-blocks)
  auto nsub = [&](int kb) { return KB - kb * SS < SS ? KB - kb * SS : SS; };   // K-blocks in slot kb
  const TcpSmem L = tcp_smem_layout(MODE, NS, ST, CS, (int)g.ldc, g.trace != nullptr, SS);
  uint8_t* ring = smem + L.ring;
  uint8_t* codes_s = smem + L.codes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L.bar);   // leader: 8 producer warps + loader tx
  uint64_t* empty_bar = full_bar + ST;                                // both: multicast MMA commit
  uint64_t* accf_bar = empty_bar + ST;                                // both: multicast MMA commit
  uint64_t* acce_bar = accf_bar + 2;                                  // leader: 2 x 8 epilogue warps
  uint64_t* codes_full = acce_bar + 2;
  uint64_t* codes_empty = codes_full + CS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem);

  const uint32_t rank = cluster_rank();
  const int pair = (int)(blockIdx.x >> 1), npair = (int)(gridDim.x >> 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int role = tcp_role(warp);
  // developer timeline of pair 0 (ITLUMM_TC_TRACE=1): slot s, event i at trace[s * kTraceEv + i];
  // slots 0/1 MMA full-wait done / ops issued, 2/3 loader of CTA 0/1 past its empty wait, 4+8r+p
  // producer warp p of CTA r arrived, 20 producer 0 of CTA 0 past its empty wait, 21 epilogue start/end
  // Stamps go to shared memory (a global store would be waited for by the producers' next proxy
  // fence and slow them down), stages [kTcpTrcFirst, +kTcpTrcWin) only; copied out at the end.
  uint64_t* trc = reinterpret_cast<uint64_t*>(smem + L.trc);
  auto stamp = [&](int slot, int64_t i) {
    if (g.trace && blockIdx.x < 2 && slot < kTcpTrcSlots && i >= kTcpTrcFirst && i < kTcpTrcFirst + kTcpTrcWin)
      trc[slot * kTcpTrcWin + (i - kTcpTrcFirst)] = clock64();   // SM cycles (cheap; %globaltimer reads are not)
  };
  // slots 16..: %globaltimer (ns, comparable across the pair's two SMs): 16 MMA full-wait done,
  // 17 / 19 producer role 0 / 7 arrived, 18 LUT loader issued (each CTA its own)
  auto stampg = [&](int slot, int64_t i) {
    if (g.trace && blockIdx.x < 2 && i >= kTcpTrcFirst && i < kTcpTrcFirst + kTcpTrcWin) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trc[slot * kTcpTrcWin + (i - kTcpTrcFirst)] = t;
    }
  };
  const int64_t ntiles = (g.N + 2 * kTcRows - 1) / (2 * kTcRows);    // 256-row pair tiles
  const int64_t units = ntiles * G;
  // k-th item of this pair: u = pair + k * npair; consecutive pairs share a slice (its LUT K-blocks
  // stream from L2 once for many pairs)
  auto item = [&](int64_t k, int64_t& tile, int& sl) -> bool {
    const int64_t u = pair + k * npair;
    if (u >= units) return false;
    sl = (int)(u / ntiles);
    tile = u - (int64_t)sl * ntiles;
    return true;
  };

  if (threadIdx.x == 0) {
    // developer: 16384 takes the producers out of the ring, 32768 the LUT loader (timing only)
    const int nfull = ((g.dbg & 16384) ? 0 : 2 * kTcpProdWarps) + ((g.dbg & 32768) ? 0 : 1);
    for (int s = 0; s < ST; ++s) { mbar_init(full_bar + s, nfull); mbar_init(empty_bar + s, 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(accf_bar + a, 1); mbar_init(acce_bar + a, 2 * kTcpEpiWarps); }
    for (int s = 0; s < CS; ++s) { mbar_init(codes_full + s, 1); mbar_init(codes_empty + s, kTcpProdWarps); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kTcpLoaderWarp && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&qt_map)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&out_map)) : "memory");
  }
  if (warp == kTcpMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(g.tmem_cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();                                   // peer barriers initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t full_leader = mapa_shared(smem_u32(full_bar), 0);
  const uint32_t acce_leader = mapa_shared(smem_u32(acce_bar), 0);
  // plan memory only above; codes and out belong to the stream order
  if (g.pdl) pdl_wait();
  pdl_launch_dependents();

  auto load_codes = [&](int64_t tile, int cs) {       // this CTA's 128-row codes tile of a pair tile
    const int64_t r0 = tile * 2 * kTcRows + (int64_t)rank * kTcRows;
    const int64_t rows = g.N - r0 < kTcRows ? (g.N - r0 > 0 ? g.N - r0 : 0) : kTcRows;
    if (rows > 0) {
      mbar_arrive_expect_tx(codes_full + cs, (uint32_t)(rows * g.ldc));
      bulk_g2s(codes_s + (size_t)cs * kTcRows * g.ldc, g.codes + r0 * g.ldc, (uint32_t)(rows * g.ldc), codes_full + cs);
    } else {
      mbar_arrive(codes_full + cs);                    // a pair tile's empty second half
    }
  };
  if (g.cload && CS > 0 && role == 18) {
    // ================================================================ codes loader (own warp): up to
    // CS items ahead of the producers, independent of the LUT ring (the LUT loader runs only ST
    // slots ahead of the MMAs, too late to hide a codes tile's L2/HBM latency at an item boundary)
    if (lane == 0) {
      int cs = 0;
      uint32_t cph = 0;
      int64_t tile;
      int sl;
      for (int64_t k = 0; item(k, tile, sl); ++k) {
        mbar_wait(codes_empty + cs, cph ^ 1);
        load_codes(tile, cs);
        if (++cs == CS) { cs = 0; cph ^= 1; }
      }
    }
  } else if (warp == kTcpLoaderWarp) {
    // ================================================================ loader (one lane per CTA)
    if (lane == 0 && !(g.dbg & 32768)) {
      const uint32_t bhalf = (uint32_t)(NS / 2) * kKBlock;
      int cs = 0, st = 0;
      uint32_t cph = 0, ph = 0;
      int64_t tile;
      int sl;
      for (int64_t k = 0; item(k, tile, sl); ++k) {
        if (!g.cload && CS > 0) {
          mbar_wait(codes_empty + cs, cph ^ 1);
          load_codes(tile, cs);
          if (++cs == CS) { cs = 0; cph ^= 1; }
        }
        const int y0 = (sl * KB) * NS + (int)rank * (NS / 2);
        for (int kb = 0; kb < KBS; ++kb) {
          mbar_wait(empty_bar + st, ph ^ 1);  // the pair's MMAs are done with the slot
          stamp(2 + (int)rank, k * KBS + kb);
          stampg(18, k * KBS + kb);
          if (g.dbg & 4) {
            if (rank == 0) mbar_arrive(full_bar + st);
          } else {
            const int ns = nsub(kb);
            if (rank == 0) mbar_arrive_expect_tx(full_bar + st, 2 * bhalf * ns);
            for (int j = 0; j < ns; ++j)
              tma_load_2d_pair(ring + (size_t)(st * SS + j) * L.stage + L.a_bytes + L.e_bytes, &qt_map, 0,
                               y0 + (kb * SS + j) * NS, full_leader + 8u * st);
          }
          if (++st == ST) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (role < kTcpProdWarps) {
    // ================================================================ producers: two threads per row
    // Thread (r, half) writes codebooks 4*half .. 4*half+3 of each 8-codebook K-block of row r.
    const int pt = role * 32 + lane;
    const int r = pt & (kTcRows - 1);
    const int half = pt >> 7;
    int cs = 0, st = 0;
    uint32_t cph = 0, ph = 0;
    int64_t tile;
    int sl;
    uint32_t doff[4];                                    // this thread's 16-byte chunks (dense layout)
#pragma unroll
    for (int j = 0; j < 4; ++j) doff[j] = sw128_off(r, 4 * half + j);
    // CS == 0: no codes tiles in shared memory (that space deepens the ring); each thread loads its
    // row's codes from global memory, 16 B per 4 K-blocks, one load ahead (across items too)
    const bool cdir = CS == 0;
    auto grow = [&](int64_t t) -> const uint8_t* {
      const int64_t rw = t * 2 * kTcRows + (int64_t)rank * kTcRows + r;
      return rw < g.N ? g.codes + rw * g.ldc : nullptr;
    };
    uint4 qnext = make_uint4(0, 0, 0, 0);
    if (cdir && item(0, tile, sl)) {
      const uint8_t* g0 = grow(tile);
      if (g0) qnext = __ldg(reinterpret_cast<const uint4*>(g0));
    }
    for (int64_t k = 0; item(k, tile, sl); ++k) {
      if (!cdir) mbar_wait(codes_full + cs, cph);
      const int64_t row = tile * 2 * kTcRows + (int64_t)rank * kTcRows + r;
      const bool valid = row < g.N;
      const uint8_t* crow = cdir ? grow(tile) : codes_s + ((size_t)cs * kTcRows + r) * g.ldc;
      const uint8_t* cnext = nullptr;                  // the next item's codes row (prefetch)
      if (cdir) {
        int64_t t2;
        int s2;
        if (item(k + 1, t2, s2)) cnext = grow(t2);
      }
      uint4 quad = make_uint4(0, 0, 0, 0);
      if (g.dbg & 16384) {
        __syncwarp();
        if (!cdir) {
          if (lane == 0) mbar_arrive(codes_empty + cs);
          if (++cs == CS) { cs = 0; cph ^= 1; }
        }
        continue;
      }
      // one ring stage per proxy fence and arrive: pairing stages made a stage wait for the NEXT
      // stage's slot to free up (one MMA pass later), which cost more than the fence it saved
      for (int kb = 0; kb < KBS; ++kb) {
#pragma unroll
        const int ns = nsub(kb);
#pragma unroll
        for (int jj = 0; jj < kTcpSsMax; ++jj) {
          if (jj >= ns) break;
          const int kbi = kb * SS + jj;
          if ((kbi & 3) == 0) {                          // 4 K-blocks of codes
            if (cdir) {
              quad = qnext;
              const uint8_t* src = kbi + 4 < KB ? (valid ? crow + (kbi + 4) * 4 : nullptr) : cnext;
              if (src) qnext = __ldg(reinterpret_cast<const uint4*>(src));
            } else if (valid) {
              quad = *reinterpret_cast<const uint4*>(crow + kbi * 4);
            }
          }
          const uint32_t cw = ((kbi & 3) == 0 ? quad.x : (kbi & 3) == 1 ? quad.y : (kbi & 3) == 2 ? quad.z : quad.w) >> (16 * half);
          const int c0 = kbi * 8 + 4 * half;               // first codebook of this thread
          const int nv = valid ? (C - c0 < 0 ? 0 : (C - c0 > 4 ? 4 : C - c0)) : 0;
          uint32_t code[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) code[j] = j < nv ? (cw >> (4 * j)) & 15u : 16u;
          if (jj == 0) mbar_wait(empty_bar + st, ph ^ 1);

          uint8_t* stg_a = ring + (size_t)(st * SS + jj) * L.stage;
          if (g.dbg & 1) {
          } else if (SP) {
            uint32_t lo[4], hi[4], m[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) onehot_sparse8(code[j], lo[j], hi[j], m[j]);
            *reinterpret_cast<uint4*>(stg_a + sw64_off(r, 2 * half)) = make_uint4(lo[0], hi[0], lo[1], hi[1]);
            *reinterpret_cast<uint4*>(stg_a + sw64_off(r, 2 * half + 1)) = make_uint4(lo[2], hi[2], lo[3], hi[3]);
            *reinterpret_cast<uint2*>(stg_a + kSpA + 16 * r + 8 * half) = make_uint2(m[0] | (m[1] << 16), m[2] | (m[3] << 16));
          } else if (g.dbg & 1024) {
            // dense, ALU-light: zero the codebook's 16 bytes, then store the single 1 byte
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              *reinterpret_cast<uint4*>(stg_a + doff[j]) = make_uint4(0, 0, 0, 0);
              if (code[j] < 16u) stg_a[doff[j] + code[j]] = 1;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint32_t w[4];
              onehot_dense16(code[j], w);
              *reinterpret_cast<uint4*>(stg_a + sw128_off(r, 4 * half + j)) = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        }
        if (!(g.dbg & 8)) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(full_leader + 8u * st);
        if (lane == 0 && rank == 0) stamp(4 + role, k * KBS + kb);
        if (lane == 0 && (role == 0 || role == 7)) stampg(role == 0 ? 17 : 19, k * KBS + kb);
        if (++st == ST) { st = 0; ph ^= 1; }
      }
      if (!cdir) {
        __syncwarp();
        if (lane == 0) mbar_arrive(codes_empty + cs);
        if (++cs == CS) { cs = 0; cph ^= 1; }
      }
    }
  } else if (warp == kTcpMmaWarp) {
    // ================================================================ MMA issuer (leader warp)
    // The whole warp runs the loop (its values stay warp-uniform, in uniform registers) and one
    // elected lane issues each tcgen05 op: a lone lane == 0 thread made the compiler move every
    // descriptor through R2UR and wrap each op in an elect loop (~190 ns per stage, tcp_trace).
    if (rank == 0) {
      const uint32_t idesc = idesc_i8_m256(NS);
      const uint32_t r0 = smem_u32(ring);
      const uint64_t a_desc0 = SP ? umma_desc_sw64(r0) : umma_desc_sw128(r0);
      const uint64_t e_desc0 = umma_desc_rows16(r0 + (uint32_t)L.a_bytes);
      const uint64_t b_desc0 = umma_desc_sw128(r0 + (uint32_t)(L.a_bytes + L.e_bytes));
      const uint32_t step = (uint32_t)(L.stage >> 4);
      const uint32_t e_col0 = tmem_base + (uint32_t)(2 * NS);
      int st = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      int64_t tile;
      int sl;
      // Issue cost per loop pass is ~270 cycles plus ~300 of loop and barrier overhead (tcp_trace),
      // more than a stage's sparse MMAs (~230 cycles): two ring stages per pass, as the producers fill
      // them.  No tcgen05.fence per stage: the smem operands are ordered by the mbarrier (TMA bytes;
      // the producers' proxy fence before their arrive); only the accumulator reuse after the
      // epilogue's tcgen05.ld needs the fence.
      auto issue = [&](int stg, int kb, uint32_t d) {
        const uint64_t ad = a_desc0 + (uint64_t)(stg * step);
        const uint64_t bd = b_desc0 + (uint64_t)(stg * step);
        if (g.dbg & 2) return;
        if (SP) {
          const uint32_t e = e_col0 + 4u * stg;
          tmem_cp_pair_128x128b(e, e_desc0 + (uint64_t)(stg * step));
          umma_sp_i8_pair(d, ad, bd, e, idesc, kb != 0);            // K = 64: codebooks 0-3
          umma_sp_i8_pair(d, ad + 2, bd + 4, e + 2, idesc, 1u);     // codebooks 4-7 (A +32 B, B +64 B)
        } else {
          umma_i8_pair(d, ad, bd, idesc, kb != 0);
          umma_i8_pair(d, ad + 2, bd + 2, idesc, 1u);
          umma_i8_pair(d, ad + 4, bd + 4, idesc, 1u);
          umma_i8_pair(d, ad + 6, bd + 6, idesc, 1u);
        }
      };
      auto issue_slot = [&](int slot, int kb, uint32_t d) {   // the SS K-blocks of one ring slot
        const int ns = nsub(kb);
#pragma unroll
        for (int j = 0; j < kTcpSsMax; ++j)
          if (j < ns) issue(slot * SS + j, kb * SS + j, d);
      };
      for (int64_t k = 0; item(k, tile, sl); ++k) {
        mbar_wait(acce_bar + acc, aph ^ 1);   // both CTAs' epilogues drained this accumulator
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * NS);
        for (int kb = 0; kb < KBS;) {
          const int st1 = st + 1 == ST ? 0 : st + 1;
          const uint32_t ph1 = st + 1 == ST ? ph ^ 1 : ph;
          mbar_wait(full_bar + st, ph);
          // the next stage too if it is already full (one issue pass for both), never wait for it
          const bool two = !(g.dbg & 4096) &&
                           __shfl_sync(0xffffffffu, (int)(kb + 1 < KBS && mbar_test(full_bar + st1, ph1)), 0) != 0;
          if (lane == 0) stamp(0, k * KBS + kb);
          if (lane == 0) stampg(16, k * KBS + kb);
          if (elect_one()) {
            issue_slot(st, kb, d);
            if (two) issue_slot(st1, kb + 1, d);
            if (g.dbg & 8192) {   // developer: free the slot by plain remote arrivals (no tensor-pipe commit)
              mbar_arrive_cluster(mapa_shared(smem_u32(empty_bar + st), 0));
              mbar_arrive_cluster(mapa_shared(smem_u32(empty_bar + st), 1));
              if (two) {
                mbar_arrive_cluster(mapa_shared(smem_u32(empty_bar + st1), 0));
                mbar_arrive_cluster(mapa_shared(smem_u32(empty_bar + st1), 1));
              }
            } else {
              umma_commit_pair(empty_bar + st);
              if (two) umma_commit_pair(empty_bar + st1);
            }
            if (kb + (two ? 2 : 1) >= KBS) umma_commit_pair(accf_bar + acc);
          }
          __syncwarp();
          if (lane == 0) stamp(1, k * KBS + kb);
          st = two ? (st1 + 1 == ST ? 0 : st1 + 1) : st1;
          ph = two ? (st1 + 1 == ST ? ph1 ^ 1 : ph1) : ph1;
          kb += two ? 2 : 1;
        }
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
  } else if (role < 16) {
    // ================================================================ epilogue (own 128 rows)
    const int e = role - kTcpProdWarps;
    const int q = warp & 3;                            // TMEM lane quadrant this warp may access
    const int h = e & 1;                              // the quadrant's two warps split the 32-column chunks
    uint8_t* stg = smem + L.stg + (size_t)e * kTcStage;
    int acc = 0;
    uint32_t aph = 0;
    const uint64_t opol = l2_policy(g.out_hint);
    bool pending = false;
    int64_t tile;
    int sl;
    for (int64_t k = 0; item(k, tile, sl); ++k) {
      mbar_wait(accf_bar + acc, aph);
      tc_fence_after();

      const int m0 = sl * NS;
      const int64_t row0 = tile * 2 * kTcRows + (int64_t)rank * kTcRows + q * 32;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * NS);
      if (row0 < g.N && !(g.dbg & 32)) {
        for (int j0 = h * 32; j0 < NS; j0 += 64) {
          uint32_t v[32];
          tmem_ld16(tbase + j0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
          tmem_ld16(tbase + j0 + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
          tmem_wait_ld();
          if (g.acc) {                                   // optional raw int32 output (tests)
            const int64_t row = row0 + lane;
            if (row < g.N) {
              int32_t* a = g.acc + row * g.ldacc + m0 + j0;
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (m0 + j0 + j < p.M) a[j] = (int32_t)v[j];
            }
          }
          if (!g.out) continue;
          float y[32];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 s4 = __ldg(reinterpret_cast<const float4*>(p.scale + m0 + j0 + 4 * c));
            const float4 o4 = __ldg(reinterpret_cast<const float4*>(p.offtot + m0 + j0 + 4 * c));
            // a4, one rounding (R8); (float)acc exactly, on the FMA pipe: acc < 2^23 (255 C < 2^23,
            // checked at plan time), so 2^23 + acc is exact and subtracting 2^23 leaves acc
            y[4 * c + 0] = fmaf(s4.x, u2f_exact(v[4 * c + 0]), o4.x);
            y[4 * c + 1] = fmaf(s4.y, u2f_exact(v[4 * c + 1]), o4.y);
            y[4 * c + 2] = fmaf(s4.z, u2f_exact(v[4 * c + 2]), o4.z);
            y[4 * c + 3] = fmaf(s4.w, u2f_exact(v[4 * c + 3]), o4.w);
          }
          if (g.relu) {
#pragma unroll
            for (int j = 0; j < 32; ++j) y[j] = relu_pos0(y[j]);
          }
          if (pending) {                                 // the previous box has left the staging
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
          }
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<float4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) =
                make_float4(y[4 * c], y[4 * c + 1], y[4 * c + 2], y[4 * c + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && !(g.dbg & 16)) {
            if (g.out_hint) tma_store_2d_hint(&out_map, stg, m0 + j0, (int)row0, opol);
            else tma_store_2d(&out_map, stg, m0 + j0, (int)row0);
            bulk_commit();
          }
          pending = !(g.dbg & 16);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acce_leader + 8u * acc);

      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
    if (lane == 0) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  if (g.trace && blockIdx.x < 2)
    for (int i = threadIdx.x; i < kTcpTrcSlots * kTcpTrcWin; i += blockDim.x) g.trace[(size_t)blockIdx.x * kTcpTrcSlots * kTcpTrcWin + i] = trc[i];
  cluster_sync_all();                                   // the pair is done with TMEM and barriers
  if (warp == kTcpMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(g.tmem_cols) : "memory");
  }
}

// ------------------------------------------------------------------------------ host side
struct TcpPlan {
  bool ok = false;
  const char* why = "not configured";
  int mode = kTcpDense;
  int KB = 0, NS = 0, G = 0, ST = 0, SS = 1, CS = 2, tmem_cols = 512;
  uint64_t* trace = nullptr;
  const uint8_t* qt = nullptr;         // [G][KB][NS][128 B] swizzled K-major LUT slices
  alignas(64) CUtensorMap qt_map;      // 2-D view, one row per (block, column); box = NS/2 rows
  int num_sms = 0;
};

// Ring depth: as many stages as fit next to 2 codes tiles of the widest rows (ldc up to
// 16 * ceil(C / 32)) and the epilogue staging, within the TMEM left by the accumulators.
inline void tcp_finish(TcpPlan& t, int C, int row_bytes) {
  t.ok = false;
  const int ldc_max = 16 * ((C + 31) / 32);
  static const int st_env = getenv("ITLUMM_TCP_STAGES") ? atoi(getenv("ITLUMM_TCP_STAGES")) : 0;   // developer
  static const int ss_env = getenv("ITLUMM_TCP_SS") ? atoi(getenv("ITLUMM_TCP_SS")) : 2;   // developer
  t.SS = ss_env < 1 ? 1 : ss_env > kTcpSsMax ? kTcpSsMax : ss_env;
  if (t.SS > t.KB) t.SS = t.KB;
  static const int cd_env = getenv("ITLUMM_TCP_CDIRECT") ? atoi(getenv("ITLUMM_TCP_CDIRECT")) : 1;   // developer
  t.CS = cd_env ? 0 : 2;   // 0: codes straight from global memory, the space goes to the ring
  int ST = 12;
  while (ST > 2 && tcp_smem_layout(t.mode, t.NS, ST, t.CS, ldc_max, false, t.SS).total > kSmemMax) --ST;
  while (t.SS > 1 && tcp_smem_layout(t.mode, t.NS, 2, t.CS, ldc_max, false, t.SS).total > kSmemMax) --t.SS;   // two slots at least
  if (st_env >= 2 && st_env < ST) ST = st_env;
  const int meta_cols = t.mode == kTcpSparse ? 4 : 0;
  if (meta_cols && 2 * t.NS + meta_cols * ST * t.SS > 512) ST = (512 - 2 * t.NS) / (meta_cols * t.SS);
  if (ST < 2) { t.why = "shared memory / TMEM budget"; return; }
  t.ST = ST;
  auto enc = tensor_map_encoder();
  if (!enc) { t.why = "no cuTensorMapEncodeTiled"; return; }
  memset(&t.qt_map, 0, sizeof t.qt_map);
  const int blocks = t.KB;
  const cuuint64_t dims[2] = {(cuuint64_t)row_bytes, (cuuint64_t)t.G * blocks * t.NS};
  const cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
  const cuuint32_t box[2] = {(cuuint32_t)row_bytes, (cuuint32_t)(t.NS / 2)};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&t.qt_map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(t.qt), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    t.why = "LUT tensor map encode failed";
    return;
  }
  cudaFuncSetAttribute((const void*)k_tcp<kTcpDense>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
  cudaFuncSetAttribute((const void*)k_tcp<kTcpSparse>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
  t.ok = true;
  t.why = "";
}

// The pair kernel over the k_tc tiling (dense or 2:4-sparse one-hot): slices NS <= 224 (sparse) or
// <= 256 (dense) columns wide, NS a multiple of 32, the LUT laid out as for k_tc (qt).
inline void tcp_configure(TcpPlan& t, const TcPlan& src, int num_sms) {
  t.ok = false;
  if (!src.ok || !src.qt) { t.why = "no tensor-core tiling"; return; }
  if (255LL * src.C >= (1LL << 23)) { t.why = "C too large for the exact 2^23 float conversion"; return; }
  if (src.NS % 32 != 0 || src.NS > (src.sp ? kTcpSpNsMax : 256)) { t.why = "slice width unsupported by the pair kernel"; return; }
  t.mode = src.sp ? kTcpSparse : kTcpDense;
  t.KB = src.KB; t.NS = src.NS; t.G = src.G; t.qt = src.qt; t.num_sms = num_sms;
  tcp_finish(t, src.C, kKBlock);
}

// Launch on codes (row-major, ldc % 16 == 0, 16-byte aligned base).  Returns EUNSUPPORTED without
// launching when those do not hold.
inline itlumm_status tcp_launch(const TcpPlan& t, const DevPlan& dp, const TcArgs& a, cudaStream_t s, bool pdl) {
  if (!t.ok) { g_tc_msg = t.why; return ITLUMM_EUNSUPPORTED; }
  if (a.ldc % 16 != 0 || (reinterpret_cast<uintptr_t>(a.codes) & 15) || (int64_t)kTcRows * a.ldc >= (1 << 20)) {
    g_tc_msg = "the pair kernel needs 16-byte aligned codes rows (ldc % 16 == 0)";
    return ITLUMM_EUNSUPPORTED;
  }
  if (!a.out && !a.acc) { g_tc_msg = "no output"; return ITLUMM_EINVAL; }
  alignas(64) CUtensorMap out_map;
  memset(&out_map, 0, sizeof out_map);
  if (a.out && !make_out_map(&out_map, a.out, a.N, dp.M, a.ldo)) {
    g_tc_msg = "output not TMA-storable (16-byte aligned base and row stride needed)";
    return ITLUMM_EUNSUPPORTED;
  }
  int CS = t.CS;
  const bool tr = t.trace != nullptr;
  if (CS > 0 && tcp_smem_layout(t.mode, t.NS, t.ST, CS, (int)a.ldc, tr, t.SS).total > kSmemMax) CS = 1;
  const size_t smem = tcp_smem_layout(t.mode, t.NS, t.ST, CS, (int)a.ldc, tr, t.SS).total;
  if (smem > kSmemMax) { g_tc_msg = "shared memory budget (codes rows too wide)"; return ITLUMM_EUNSUPPORTED; }
  TcpKArgs k{};
  k.codes = a.codes; k.ldc = a.ldc; k.N = a.N; k.acc = a.acc; k.ldacc = a.ldacc; k.out = a.out; k.ldo = a.ldo;
  k.relu = a.relu; k.KB = t.KB; k.NS = t.NS; k.G = t.G; k.ST = t.ST; k.SS = t.SS; k.CS = CS; k.tmem_cols = t.tmem_cols;
  k.pdl = pdl ? 1 : 0;
  k.trace = t.trace;
  static const int dbg = getenv("ITLUMM_TCP_DBG") ? atoi(getenv("ITLUMM_TCP_DBG")) : 0;   // developer
  k.dbg = dbg;
  static const int cl_env = getenv("ITLUMM_TCP_CLOAD") ? atoi(getenv("ITLUMM_TCP_CLOAD")) : 1;   // developer
  k.cload = cl_env;
  // Output stores carry L2 evict_first when the call's output is far larger than the L2 (> 1 GB: cfg5's
  // 4.3 GB, cfg4's hidden layers), so that the stream does not push codes and LUT out: k_tcp 3.14 -> 3.09 ms
  // at cfg5.  Smaller outputs keep the default policy: with the hint the row-major cfg3 step ran 154 -> 160
  // us although both kernels alone were no slower (the write-back then competes with the next call's
  // HBM-bound row encoder).  Developer override: ITLUMM_OUT_HINT (l2_policy kind).
  static const int oh_env = getenv("ITLUMM_OUT_HINT") ? atoi(getenv("ITLUMM_OUT_HINT")) : -1;
  k.out_hint = oh_env >= 0 ? oh_env : ((unsigned long long)a.N * (unsigned long long)dp.M * 4ull > (1ull << 30) ? 1 : 0);
  const int64_t units = ((a.N + 255) / 256) * t.G;
  const void* kfn = t.mode == kTcpSparse ? (const void*)k_tcp<kTcpSparse> : (const void*)k_tcp<kTcpDense>;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kTcpThreads);
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
  cfg.numAttrs = 1;
  // Persistent: exactly as many pairs as can be co-resident (a GPC with an odd number of free SMs
  // leaves one idle), so that no pair runs in a second wave behind the others.
  int max_clusters = 0;
  cfg.gridDim = dim3((unsigned)(t.num_sms / 2 * 2));
  if (cudaOccupancyMaxActiveClusters(&max_clusters, kfn, &cfg) != cudaSuccess || max_clusters < 1) {
    cudaGetLastError();
    max_clusters = t.num_sms / 2;
  }
  int64_t pairs = max_clusters < t.num_sms / 2 ? max_clusters : t.num_sms / 2;
  if (pairs > units) pairs = units;
  cfg.gridDim = dim3((unsigned)(2 * pairs));
  cfg.numAttrs = pdl ? 2 : 1;
  cudaError_t e = t.mode == kTcpSparse ? cudaLaunchKernelEx(&cfg, k_tcp<kTcpSparse>, dp, k, out_map, t.qt_map)
                                       : cudaLaunchKernelEx(&cfg, k_tcp<kTcpDense>, dp, k, out_map, t.qt_map);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) { g_tc_msg = cudaGetErrorString(e); return ITLUMM_ECUDA; }
  return ITLUMM_OK;
}

}  // namespace itlumm
