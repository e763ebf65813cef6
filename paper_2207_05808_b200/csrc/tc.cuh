// tc.cuh — tcgen05 one-hot x LUT tensor-core kernel.
//
// The lookup-accumulate a3 is the product G.Q of the one-hot encoding G (N x 16C, "the
// concatenation of C one-hot 16-dimensional vectors") with the uint8 LUT Q (16C x M):
// acc = G.Q exactly, then the a4 epilogue.  Per persistent CTA:
//   producer warps  : FUSED: gather the 4C split columns of each row and walk the trees (a1+a2);
//                     else: read nibble-packed codes.  Either way they write the one-hot tile
//                     (128 rows x 128 B = 8 codebooks per K-block) straight into shared memory
//                     in the UMMA canonical K-major SWIZZLE_128B layout (one 16-byte chunk per
//                     (row, codebook)), ring of SA K-block stages.
//   MMA warp        : one elected thread issues tcgen05.mma.cta_group::1.kind::i8 (u8 x u8 -> s32,
//                     M=128, N=NS, K=32 per instruction = 2 codebooks) into a TMEM accumulator
//                     (double buffered), B = the CTA's LUT slice, resident in shared memory.
//   epilogue warps  : tcgen05.ld the s32 accumulators, y = fmaf(scale, (float)acc, offtot) (+ReLU),
//                     store fp32 rows.
// Integer products/sums of u8 one-hot x u8 LUT are exact, so results equal the SIMT path bit for bit.
#pragma once
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "../../include/itlumm.h"
#include "common.cuh"

namespace itlumm {

constexpr int kTcProducerWarps = 4;
constexpr int kTcProducers = 32 * kTcProducerWarps;           // one producer thread per tile row
constexpr int kTcMmaWarp = kTcProducerWarps;                   // warp 4
constexpr int kTcEpiWarp0 = kTcProducerWarps + 1;              // warps 5..12
constexpr int kTcEpiWarps = 8;                                 // 2 per TMEM lane quadrant
constexpr int kTcEpiThreads = 32 * kTcEpiWarps;
constexpr int kTcLoaderWarp = kTcEpiWarp0 + kTcEpiWarps;       // warp 13: codes bulk loads
constexpr int kTcThreads = 32 * (kTcProducerWarps + 1 + kTcEpiWarps + 1);   // 448
constexpr int kTcRows = 128;                                   // UMMA M
constexpr int kKBlock = 128;                                   // bytes of K per block = 8 codebooks
constexpr int kTcStages = 3;                                   // default A ring depth (K-blocks)
constexpr size_t kTcBBudget = 128 * 1024;                      // resident LUT slice budget
constexpr int kTcStage = 32 * 32 * 4;                          // epilogue staging per warp (bytes)
constexpr size_t kSmemMax = 227 * 1024;                        // dynamic shared memory per CTA
// 2:4-sparse one-hot (f2): a one-hot 16-vector has one nonzero per 4 groups of 4, so it is 2:4
// sparse; stored compressed (2 of every 4 K-elements: 8 B per codebook) with 4 bits of metadata
// per group, tcgen05.mma.sp doubles K per instruction (K = 64 = 4 codebooks).
constexpr int kSpA = kTcRows * kKBlock / 2;                    // compressed K-block: 128 rows x 64 B, SWIZZLE_64B
constexpr int kSpStage = kSpA + kTcRows * 16;                  // + 16 B of metadata per row (tcgen05.cp source)
constexpr int kSpNsMax = 224;                                  // 2 x NS accumulators + 4 metadata columns per stage <= 512

struct TcPlan {
  bool ok = false;
  const char* why = "not configured";
  const uint8_t* qt = nullptr;   // device: [G][KB][NS][128] swizzled K-major LUT slices
  int C = 0, M = 0, KB = 0, NS = 0, G = 0, tmem_cols = 0;
  int CS = 0;                    // codes ring stages (TMA path), 0 = codes path unavailable
  bool stream_b = false;         // LUT too large to stay resident: B K-blocks streamed per stage
  bool sp = false;               // 2:4-sparse one-hot (tcgen05.mma.sp), NS <= kSpNsMax
  int ST = kTcStages;            // ring stages (one-hot K-blocks, + LUT K-blocks when streamed)
  uint64_t* trace = nullptr;     // developer timeline buffer (ITLUMM_TC_TRACE=1), 8 x 4 x kTraceEv
  size_t smem = 0;
  int grid = 0;
};

struct TcArgs {
  const void* A; int64_t lda; const uint8_t* codes; int64_t ldc; int64_t N;
  int32_t* acc; int64_t ldacc; float* out; int64_t ldo; int relu;
  int packed = 0;  // fused: split-packed rows (gather column of (c, t) is 4c + t) with 16-B aligned rows
};

struct TcKArgs {
  const void* A; int64_t lda;
  const uint8_t* codes; int64_t ldc;
  int64_t N;
  int32_t* acc; int64_t ldacc;
  float* out; int64_t ldo;
  int relu;
  int packed;      // fused producers: split-packed rows, one vector load per codebook
  int a_tma;       // fused, resident LUT, f32 split-packed rows: the loader warp stages each K-block's
                   // 128 rows x 32 floats by TMA (a_map, SWIZZLE_128B) into the one-hot stage itself
  const uint8_t* qt;
  int KB, NS, G, tmem_cols;
  int CS;          // codes ring stages; > 0 selects the bulk-copy (TMA) codes path
  int pdl;         // launched as a programmatic dependent of the encode kernel
  int tma_store;   // out written by TMA tensor stores through out_map (else per-thread stores)
  // streamed-B mode (LUT larger than shared memory, codes path only): work items are
  // (row tile, slice) pairs u = cta + k * ncta, slice = u / ntiles (consecutive CTAs share a slice,
  // so its K-blocks stream from L2); each stage carries the one-hot K-block and the LUT K-block.
  int stream_b;
  int ST;          // ring stages
  int out_hint;    // L2 policy of the output tensor stores (l2_policy kind; 0 = default)
  int dbg;         // developer removal switches (ITLUMM_TC_DBG; results then wrong): 1 producers skip
                   // the one-hot stores, 2 no MMAs (commits only), 4 no LUT copies, 16 epilogue
                   // skips the output stores, 32 no epilogue work
  uint64_t* trace; // developer timeline (ITLUMM_TC_TRACE): [8 CTAs][4 roles][kTraceEv] globaltimer stamps
};
constexpr int kTraceEv = 512;
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// TMA tensor store of one 32x32 fp32 box (128-byte swizzled rows in shared memory) at (x=col, y=row);
// rows >= N and columns >= M are clipped by the tensor map bounds.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(src)), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, const void* src, int x, int y, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(src)), "r"(x), "r"(y), "l"(pol) : "memory");
}
// TMA tensor load of one box at (x, y) into shared memory, completing on `mbar`
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* mbar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(mbar)) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SMEM matrix descriptor: K-major, SWIZZLE_128B, 8-row atoms of 1024 B (SBO), LBO unused (1),
// version 1 (sm_100), base offset 0 (atoms are 1024-byte aligned).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// Instruction descriptor, kind::i8: D s32, A u8, B u8, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kTcRows >> 4) << 24);
}
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// K-major SWIZZLE_64B (8-row atoms of 512 B): the compressed sparse one-hot.
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
// Unswizzled 128 rows x 16 B (8-row core groups 128 B apart): the tcgen05.cp metadata source.
__device__ __forceinline__ uint64_t umma_desc_rows16(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(128 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// 2:4-sparse A (bit 2 of the instruction descriptor), metadata at TMEM address e.
__device__ __forceinline__ void umma_sp_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t tmem_e,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%3], %4, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(tmem_e), "r"(idesc | 4u), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_cp_128x128b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Byte offset of the 16-byte chunk j (0..7) of row r in a K-major SWIZZLE_128B tile.
__host__ __device__ __forceinline__ uint32_t sw128_off(uint32_t r, uint32_t j) {
  return (r >> 3) * 1024u + (r & 7u) * 128u + ((j ^ (r & 7u)) << 4);
}

// Byte offset of the 16-byte chunk j (0..3) of row r in a K-major SWIZZLE_64B tile.
__host__ __device__ __forceinline__ uint32_t sw64_off(uint32_t r, uint32_t j) {
  return (r >> 3) * 512u + (r & 7u) * 64u + ((j ^ ((r >> 1) & 3u)) << 4);
}

// One row's one-hot K-block (8 codebooks; code 16 = none) into A stage `st`.
// Dense: 16 B per codebook, byte `code` = 1 (SWIZZLE_128B).  Sparse (2:4): 8 B per codebook, group
// g = code >> 2 holds the pair of logical positions (e, 3) with values (1, 0) for e = code & 3 < 3,
// or (0, 3) with values (0, 1) for e = 3; metadata nibble g = idx0 | idx1 << 2, the three empty
// groups (0, 0) with zero values; the row's 128 metadata bits (codebook j at bits 16j..16j+15)
// go to the stage's metadata rows.
template <bool SP>
__device__ __forceinline__ void put_onehot(uint8_t* st, int r, const uint32_t (&code)[8]) {
  if (!SP) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t k = code[j];
      const uint32_t bit = (k < 16) ? (1u << ((k & 3u) * 8u)) : 0u;
      const uint32_t w = k >> 2;
      *reinterpret_cast<uint4*>(st + sw128_off(r, j)) =
          make_uint4(w == 0 ? bit : 0u, w == 1 ? bit : 0u, w == 2 ? bit : 0u, w == 3 ? bit : 0u);
    }
  } else {
    uint32_t meta[4];
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      uint32_t v[2][2], m = 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t k = code[2 * jj + h];
        const uint32_t e = k & 3u, grp = (k >> 2) & 3u;
        const uint32_t idx = 2u * grp + (e == 3u ? 1u : 0u);     // stored byte of the codebook's 8
        const uint32_t bit = (k < 16) ? (1u << (8u * (idx & 3u))) : 0u;
        v[h][0] = idx < 4 ? bit : 0u;
        v[h][1] = idx < 4 ? 0u : bit;
        if (k < 16) m |= (0xCu | (e == 3u ? 0u : e)) << (4u * grp + 16u * h);
      }
      meta[jj] = m;
      *reinterpret_cast<uint4*>(st + sw64_off(r, jj)) = make_uint4(v[0][0], v[0][1], v[1][0], v[1][1]);
    }
    *reinterpret_cast<uint4*>(st + kSpA + 16 * r) = make_uint4(meta[0], meta[1], meta[2], meta[3]);
  }
}

// Shared-memory carve-up (offsets from a 1024-aligned base).
struct TcSmem {
  size_t b, a, stg, codes, thr, cols, sc, ot, bar, tmem, total;
};
// CS codes stages of 128 rows x ldc_tma bytes (the TMA codes path; CS = 0 when unused).
// stream_b: no resident slice; each of the kTcStages stages holds a one-hot K-block and a LUT
// K-block (NS x 128 B).  fused = false: no threshold/column tables.
__host__ __device__ inline TcSmem tc_smem_layout(int C, int KB, int NS, int CS = 0, int ldc_tma = 0,
                                                 bool stream_b = false, bool fused = true, int ST = kTcStages,
                                                 bool sp = false) {
  TcSmem s{};
  size_t o = 0;
  s.b = o;    o += stream_b ? (size_t)ST * NS * kKBlock : (size_t)KB * NS * kKBlock;
  s.a = o;    o += (size_t)ST * (sp ? kSpStage : kTcRows * kKBlock);   // both multiples of 1024
  s.stg = o;  o += (size_t)kTcEpiWarps * kTcStage;
  s.codes = o; o += (size_t)CS * kTcRows * ldc_tma;
  if (!fused) C = 0;
  s.thr = o;  o += (size_t)C * 16 * 4;          // thresholds [C][16] (15 used)
  s.cols = o; o += (size_t)C * 16;              // cols [C][4]
  s.sc = o;   o += (size_t)NS * 4;
  s.ot = o;   o += (size_t)NS * 4;
  o = (o + 7) & ~(size_t)7;
  s.bar = o;  o += (size_t)(3 * ST + 4 + 2 * CS + (stream_b ? 1 : KB)) * 8;   // + ST a_full (fused TMA rows)
  s.tmem = o; o += 16;
  s.total = o + 1024;                           // slack for 1024-byte alignment of the base
  return s;
}

// One persistent CTA of the tensor-core kernel: CTA `cta` of `ncta` (slice = cta % G).
template <bool FUSED, typename T, bool SB, bool SP = false>
__device__ __forceinline__ void tc_cta(const DevPlan& p, const TcKArgs& g, const CUtensorMap* out_map,
                                       const CUtensorMap* a_map, uint8_t* smem_raw, int cta, int ncta) {
  // align in the shared window without leaving the shared address space (keeps LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int C = p.C, KB = g.KB, NS = g.NS, G = g.G;
  const int CS = FUSED ? 0 : g.CS;
  const int ST = g.ST;                                // A (and streamed-B) ring depth
  const TcSmem L = tc_smem_layout(C, KB, NS, CS, (int)g.ldc, SB, FUSED, ST, SP);
  constexpr int kAStage = SP ? kSpStage : kTcRows * kKBlock;
  uint8_t* b_s = smem + L.b;
  uint8_t* codes_s = smem + L.codes;
  uint8_t* a_s = smem + L.a;
  float* thr_s = reinterpret_cast<float*>(smem + L.thr);
  int32_t* cols_s = reinterpret_cast<int32_t*>(smem + L.cols);
  float* sc_s = reinterpret_cast<float*>(smem + L.sc);
  float* ot_s = reinterpret_cast<float*>(smem + L.ot);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* empty_bar = full_bar + ST;
  uint64_t* accf_bar = empty_bar + ST;
  uint64_t* acce_bar = accf_bar + 2;
  uint64_t* codes_bar = acce_bar + 2;
  uint64_t* codes_empty = codes_bar + CS;            // producers done with a codes stage
  uint64_t* b_bar = codes_empty + CS;                // resident LUT slice: K-block kb landed (b_bar[kb])
  uint64_t* afull_bar = b_bar + (SB ? 1 : KB);        // fused TMA rows: the stage's A rows landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem);

  const int slice = cta % G;
  const int group = cta / G;
  const int ngroups = ncta / G;
  const int64_t ntiles = (g.N + kTcRows - 1) / kTcRows;
  // k-th work item of this CTA: (row tile, slice); false when the CTA is done
  // Work balance: whole (tile, slice) items first, `full` rounds of them; the `rem` leftover items
  // of the last round are split into `parts` column ranges (of the NC 32-column epilogue chunks)
  // spread over the idle CTAs, so no CTA runs a whole extra tile while the others idle (the
  // epilogue is the per-tile bottleneck; cfg2: 469 tiles on 74 CTA pairs = 6.34 rounds).
  const int NC = NS / 32;
  const int64_t units = SB ? ntiles * G : ntiles;       // items sharing this CTA's slice set
  const int64_t nworkers = SB ? ncta : ngroups;
  const int64_t worker = SB ? cta : group;
  const int64_t full = units / nworkers, rem = units - full * nworkers;
  int parts = 1;
  if (rem) {
    const int64_t pp = nworkers / rem;
    parts = pp < 1 ? 1 : (pp > NC ? NC : (int)pp);
  }
  auto item4 = [&](int64_t k, int64_t& tile, int& sl, int& c0, int& c1) -> bool {
    int64_t u;
    c0 = 0;
    c1 = NC;
    if (k < full) {
      u = worker + k * nworkers;
    } else if (k == full && worker < rem * parts) {
      u = full * nworkers + worker / parts;
      const int part = (int)(worker % parts);
      c0 = part * NC / parts;
      c1 = (part + 1) * NC / parts;
    } else {
      return false;
    }
    if (SB) {
      sl = (int)(u / ntiles);
      tile = u - (int64_t)sl * ntiles;
    } else {
      sl = slice;
      tile = u;
    }
    return true;
  };
  auto item = [&](int64_t k, int64_t& tile, int& sl) -> bool {
    int c0, c1;
    return item4(k, tile, sl, c0, c1);
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* trace = (g.trace && cta < 8) ? g.trace + (size_t)cta * 4 * kTraceEv : nullptr;
  // per-CTA spans after the role timelines: [16 x 4 x kTraceEv] | encoder [512][2] | TC [512][2]
  uint64_t* span = (g.trace && cta < 512) ? g.trace + (size_t)16 * 4 * kTraceEv + 2 * 512 + 2 * cta : nullptr;
  if (span && threadIdx.x == 0) span[0] = gtimer();
  int tev[4] = {0, 0, 0, 0};
  auto stamp = [&](int role) {                          // role: 0 producer, 1 MMA, 2 epilogue, 3 loader
    if (trace && tev[role] < kTraceEv) trace[role * kTraceEv + tev[role]++] = gtimer();
  };

  // ---- prologue: the resident LUT slice (already swizzled in HBM) by bulk copy (TMA engine),
  // thresholds, columns, scales by the threads; only the MMA warp waits for the slice.
  {
    if (threadIdx.x == 0 && !SB) {
      // one barrier per K-block (NS x 128 B <= 32 KB): the first item's MMAs start on K-block 0
      // while the rest of the slice is still landing
      for (int kb = 0; kb < KB; ++kb) mbar_init(b_bar + kb, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      const uint8_t* src = g.qt + (size_t)slice * KB * NS * kKBlock;
      const uint32_t blk = (uint32_t)NS * kKBlock;
      for (int kb = 0; kb < KB; ++kb) {
        mbar_arrive_expect_tx(b_bar + kb, blk);
        bulk_g2s(b_s + (size_t)kb * blk, src + (size_t)kb * blk, blk, b_bar + kb);
      }
    }
    if (FUSED) {
      for (int i = threadIdx.x; i < C * 16; i += blockDim.x) {
        const int c = i >> 4, h = i & 15;
        thr_s[i] = h < 15 ? __ldg(p.thr_t + h * C + c) : 0.f;
      }
      for (int i = threadIdx.x; i < 4 * C; i += blockDim.x) cols_s[i] = __ldg(p.cols + i);
    }
    for (int i = threadIdx.x; i < NS && !SB; i += blockDim.x) {
      const int m = slice * NS + i;
      sc_s[i] = m < p.Mp ? __ldg(p.scale + m) : 0.f;
      ot_s[i] = m < p.Mp ? __ldg(p.offtot + m) : 0.f;
    }
    if (threadIdx.x == 0) {
      for (int s = 0; s < ST; ++s) { mbar_init(full_bar + s, kTcProducers + (SB ? 1 : 0)); mbar_init(empty_bar + s, 1); mbar_init(afull_bar + s, 1); }
      for (int a = 0; a < 2; ++a) { mbar_init(accf_bar + a, 1); mbar_init(acce_bar + a, kTcEpiThreads); }
      for (int s = 0; s < CS; ++s) { mbar_init(codes_bar + s, 1); mbar_init(codes_empty + s, kTcProducers); }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kTcMmaWarp) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(g.tmem_cols) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  const uint32_t tmem_base = *tmem_slot;
  // Everything above touched only plan memory; the codes (and `out`) belong to the stream
  // order, so a programmatic dependent waits here for the encode grid to complete.
  if (g.pdl) pdl_wait();
  pdl_launch_dependents();           // a programmatically dependent next encoder may start its prologue

  if (warp == kTcLoaderWarp) {
    // ============================================================== codes loader (one lane)
    // Codes tiles (128 rows x ldc bytes, contiguous) through a CS-deep bulk-copy ring (when the
    // codes rows can be bulk-copied), and with a streamed LUT (SB) the item's LUT K-blocks.
    if (lane == 0 && FUSED && !SB && g.a_tma) {
      // fused, split-packed f32 rows: K-block kb of a tile is the box (x = 32 kb, y = 128 tile) of
      // 128 rows x 128 B, loaded into the one-hot stage the producers then overwrite in place
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(a_map)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      int64_t tile;
      int sl;
      for (int64_t k = 0; item(k, tile, sl); ++k) {
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(empty_bar + stage, phase ^ 1);    // MMA finished reading this stage
          mbar_arrive_expect_tx(afull_bar + stage, (uint32_t)(kTcRows * kKBlock));
          tma_load_2d(a_s + (size_t)stage * kAStage, a_map, 32 * kb, (int)(tile * kTcRows), afull_bar + stage);
          stamp(3);
          if (++stage == ST) { stage = 0; phase ^= 1; }
        }
      }
    } else if (lane == 0 && ((!FUSED && CS > 0) || SB)) {
      int cs = 0, stage = 0;
      uint32_t cph = 0, phase = 0;
      int64_t tile;
      int sl;
      for (int64_t k = 0; item(k, tile, sl); ++k) {
        if (!FUSED && CS > 0) {
          mbar_wait(codes_empty + cs, cph ^ 1);
          const int64_t r0 = tile * kTcRows;
          const int rows = (int)((g.N - r0) < kTcRows ? (g.N - r0) : (int64_t)kTcRows);
          const uint32_t bytes = (uint32_t)(rows * g.ldc);
          mbar_arrive_expect_tx(codes_bar + cs, bytes);
          bulk_g2s(codes_s + (size_t)cs * kTcRows * g.ldc, g.codes + r0 * g.ldc, bytes, codes_bar + cs);
          stamp(3);
          if (++cs == CS) { cs = 0; cph ^= 1; }
        }
        if (SB) {                                     // this item's LUT K-blocks, one per stage
          const uint32_t bbytes = (uint32_t)NS * kKBlock;
          const uint8_t* src = g.qt + (size_t)sl * KB * bbytes;
          for (int kb = 0; kb < KB; ++kb) {
            mbar_wait(empty_bar + stage, phase ^ 1);
            if (g.dbg & 4) {
              mbar_arrive(full_bar + stage);
            } else {
              mbar_arrive_expect_tx(full_bar + stage, bbytes);
              bulk_g2s(b_s + (size_t)stage * bbytes, src + (size_t)kb * bbytes, bbytes, full_bar + stage);
            }
            stamp(3);
            if (++stage == ST) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else

  if (warp < kTcProducerWarps) {
    // ============================================================== producers: one row each
    // The input of K-block i+1 (32 gathered values, or 4 code bytes) is loaded before K-block i
    // is encoded and written, so one K-block of loads is always in flight per thread.
    const int r = threadIdx.x;                       // row within the tile, 0..127
    if (!FUSED && CS > 0) {
      // Codes arrive by bulk copy (loader warp), CS tiles ahead; each producer thread reads its
      // row's 4 code bytes per K-block from shared memory and writes 8 one-hot chunks.
      int stage = 0, cs = 0;
      uint32_t phase = 0, cph = 0;
      int64_t tile;
      int sl;
      for (int64_t kk = 0; item(kk, tile, sl); ++kk) {
        mbar_wait(codes_bar + cs, cph);
        const bool valid = tile * kTcRows + r < g.N;
        const uint8_t* crow = codes_s + ((size_t)cs * kTcRows + r) * g.ldc;
        uint4 quad = make_uint4(0, 0, 0, 0);
        for (int kb = 0; kb < KB; ++kb) {
          // one 16-byte read per 4 K-blocks: a 4-byte read per K-block of rows ldc apart was a
          // 32-way bank conflict when ldc is a multiple of 128 (cfg5; ncu r02)
          if ((kb & 3) == 0 && valid) quad = *reinterpret_cast<const uint4*>(crow + kb * 4);
          const uint32_t cw = (kb & 3) == 0 ? quad.x : (kb & 3) == 1 ? quad.y : (kb & 3) == 2 ? quad.z : quad.w;
          uint32_t code[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) code[j] = (valid && kb * 8 + j < C) ? (cw >> (4 * j)) & 15u : 16u;
          mbar_wait(empty_bar + stage, phase ^ 1);    // MMA finished reading this stage
          if (!(g.dbg & 1)) put_onehot<SP>(a_s + (size_t)stage * kAStage, r, code);
          fence_proxy_async_smem();
          mbar_arrive(full_bar + stage);
          if (r == 0) stamp(0);
          if (++stage == ST) { stage = 0; phase ^= 1; }
        }
        mbar_arrive(codes_empty + cs);                 // this producer is done with stage cs
        if (++cs == CS) { cs = 0; cph ^= 1; }
      }
    } else if (FUSED && !SB && !SP && g.a_tma) {
      // Row r's 8 codebooks x 4 split values landed by TMA as row r of the stage (chunk j of the
      // 128 B at 16 (j ^ (r & 7)), SWIZZLE_128B: conflict-free reads); the thread walks the 8 trees
      // and overwrites exactly those 128 B with its one-hot row (the same swizzled chunks).
      int stage = 0;
      uint32_t phase = 0;
      int64_t tile;
      int sl;
      for (int64_t kk = 0; item(kk, tile, sl); ++kk) {
        const bool valid = tile * kTcRows + r < g.N;
        for (int kb = 0; kb < KB; ++kb) {
          uint8_t* st = a_s + (size_t)stage * kAStage;
          mbar_wait(afull_bar + stage, phase);
          float4 q[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) q[j] = *reinterpret_cast<const float4*>(st + sw128_off(r, j));
          uint32_t code[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int c = kb * 8 + j;
            code[j] = 16;
            if (valid && c < C) {
              const float* th = thr_s + c * 16;
              const float vv[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
              int node = 0;
#pragma unroll
              for (int t = 0; t < kLevels; ++t) node = 2 * node + (vv[t] > th[(1 << t) - 1 + node] ? 1 : 0);
              code[j] = (uint32_t)node;
            }
          }
          put_onehot<false>(st, r, code);
          fence_proxy_async_smem();
          mbar_arrive(full_bar + stage);
          if (r == 0) stamp(0);
          if (++stage == ST) { stage = 0; phase ^= 1; }
        }
      }
    } else {
    const bool codes_u32 = !FUSED && ((g.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(g.codes) & 3) == 0);
    int stage = 0;
    uint32_t phase = 0;
    float vc[8][4], vn[8][4];
    uint32_t cc = 0, cn = 0;
    auto load = [&](int64_t tile, int kb, float (&v)[8][4], uint32_t& cw) {
      const int64_t row = tile * kTcRows + r;
      if (row >= g.N) return;
      if (FUSED && g.packed) {
        // split-packed row: codebook c's four split values are a[4c..4c+3], one 16-byte (f32) or
        // 8-byte (bf16) load each; the 8 loads of a K-block cover 128 (64) contiguous bytes
        const T* a = reinterpret_cast<const T*>(g.A) + row * g.lda;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = kb * 8 + j;
          if (c < C) {
            if (sizeof(T) == 4) {
              const float4 q = __ldg(reinterpret_cast<const float4*>(a + 4 * c));
              v[j][0] = q.x; v[j][1] = q.y; v[j][2] = q.z; v[j][3] = q.w;
            } else {
              const uint2 q = __ldg(reinterpret_cast<const uint2*>(a + 4 * c));
              v[j][0] = __uint_as_float(q.x << 16); v[j][1] = __uint_as_float(q.x & 0xFFFF0000u);
              v[j][2] = __uint_as_float(q.y << 16); v[j][3] = __uint_as_float(q.y & 0xFFFF0000u);
            }
          }
        }
      } else if (FUSED) {
        const T* a = reinterpret_cast<const T*>(g.A) + row * g.lda;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = kb * 8 + j;
          if (c < C) {
            const int4 col = *reinterpret_cast<const int4*>(cols_s + 4 * c);
            v[j][0] = InTraits<T>::load(a + col.x);
            v[j][1] = InTraits<T>::load(a + col.y);
            v[j][2] = InTraits<T>::load(a + col.z);
            v[j][3] = InTraits<T>::load(a + col.w);
          }
        }
      } else {
        const uint8_t* cp = g.codes + row * g.ldc + kb * 4;
        const int nbytes = ((C + 1) >> 1) - kb * 4;      // valid code bytes from this K-block
        if (codes_u32 && nbytes >= 4) {
          cw = __ldg(reinterpret_cast<const unsigned int*>(cp));
        } else {
          cw = 0;
          for (int b = 0; b < 4 && b < nbytes; ++b) cw |= (uint32_t)__ldg(cp + b) << (8 * b);
        }
      }
    };
    // the same item sequence as the MMA and epilogue warps (including split leftover items)
    int64_t k = 0, tile = 0;
    int sl = 0, kb = 0;
    bool more = item(0, tile, sl);
    if (more) load(tile, 0, vc, cc);
    while (more) {
      int64_t ntile = tile, nk = k;
      int nkb = kb + 1;
      bool nmore = true;
      if (nkb == KB) { nkb = 0; ++nk; nmore = item(nk, ntile, sl); }
      if (nmore) load(ntile, nkb, vn, cn);
      const bool valid = tile * kTcRows + r < g.N;
      uint32_t code[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = kb * 8 + j;
        code[j] = 16;                                   // 16 = no one-hot bit (padding)
        if (valid && c < C) {
          if (FUSED) {
            const float* th = thr_s + c * 16;
            int node = 0;
#pragma unroll
            for (int t = 0; t < kLevels; ++t) node = 2 * node + (vc[j][t] > th[(1 << t) - 1 + node] ? 1 : 0);
            code[j] = (uint32_t)node;
          } else {
            code[j] = (cc >> (4 * j)) & 15u;
          }
        }
      }
      mbar_wait(empty_bar + stage, phase ^ 1);        // MMA finished reading this stage
      put_onehot<SP>(a_s + (size_t)stage * kAStage, r, code);
      fence_proxy_async_smem();
      mbar_arrive(full_bar + stage);
      if (++stage == ST) { stage = 0; phase ^= 1; }
      if (FUSED) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
          for (int t = 0; t < 4; ++t) vc[j][t] = vn[j][t];
      } else {
        cc = cn;
      }
      tile = ntile;
      kb = nkb;
      k = nk;
      more = nmore;
    }
    }
  } else if (warp == kTcMmaWarp) {
    // ============================================================== MMA issuer
    // One thread, kept lean: the tensor core only stays busy if the issuing thread turns a K-block
    // around in less than its MMA time (272 ns at N=256); descriptors are precomputed and advanced
    // by adding to the start-address field (addr >> 4; shared addresses < 256 KB never carry).
    {
      // the whole warp runs the loop (warp-uniform values stay in uniform registers), one elected
      // lane issues each tcgen05 op (a lone lane == 0 thread wrapped every op in an elect loop and
      // moved every descriptor through R2UR: ~190 ns per stage in the k_tcp timeline, profiles/r02)
      const uint32_t idesc = idesc_i8(NS);
      const uint32_t a0 = smem_u32(a_s);
      const uint64_t a_desc0 = SP ? umma_desc_sw64(a0) : umma_desc_sw128(a0);
      const uint64_t m_desc0 = umma_desc_rows16(a0 + kSpA);
      const uint64_t b_desc0 = umma_desc_sw128(smem_u32(b_s));
      const uint32_t a_step = (uint32_t)kAStage >> 4, b_step = (uint32_t)(NS * kKBlock) >> 4;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int64_t tile;
      int sl;
      for (int64_t k = 0; item(k, tile, sl); ++k) {
        mbar_wait(acce_bar + acc, acc_phase ^ 1);    // epilogue drained this accumulator
        if (lane == 0) stamp(1);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * NS);
        for (int kb = 0; kb < KB; ++kb) {
          if (!SB && k == 0) mbar_wait(b_bar + kb, 0);   // the resident LUT slice's K-block kb
          mbar_wait(full_bar + stage, phase);
          const uint64_t ad = a_desc0 + (uint64_t)(stage * a_step);
          const uint64_t bd = b_desc0 + (uint64_t)((SB ? stage : kb) * b_step);
          if (elect_one()) {
            if (g.dbg & 2) {
            } else if (SP) {
              // metadata rows -> TMEM columns 2NS + 4*stage (in tcgen05 issue order before the MMAs
              // that read them), then 2 sparse MMAs of K = 64 (4 codebooks each; A +32 B, B +64 B)
              const uint32_t e = tmem_base + (uint32_t)(2 * NS + 4 * stage);
              tmem_cp_128x128b(e, m_desc0 + (uint64_t)(stage * a_step));
              umma_sp_i8(d, ad, bd, e, idesc, kb != 0);
              umma_sp_i8(d, ad + 2, bd + 4, e + 2, idesc, 1u);
            } else {
              umma_i8(d, ad, bd, idesc, kb != 0);          // K = 32 per MMA: +32 B on both operands
              umma_i8(d, ad + 2, bd + 2, idesc, 1u);
              umma_i8(d, ad + 4, bd + 4, idesc, 1u);
              umma_i8(d, ad + 6, bd + 6, idesc, 1u);
            }
            umma_commit(empty_bar + stage);             // frees the stage when these MMAs finish
            if (kb == KB - 1) umma_commit(accf_bar + acc);
          }
          __syncwarp();
          if (lane == 0) stamp(1);
          if (++stage == ST) { stage = 0; phase ^= 1; }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ============================================================== epilogue
    // Warp e covers TMEM lane quadrant q (rows 32q..32q+31) and the 32-column chunks j0 = 32h,
    // 32h+64, ... (h = e / 4).  Per chunk: tcgen05.ld the raw s32 accumulators of its 32 rows,
    // stage them row-major (16-byte slots XOR-swizzled by row) in shared memory, then each lane
    // reads back 4 consecutive columns of one row, dequantises them with its register-resident
    // scale/offtot (a4: one fmaf per element, R8; ReLU R9) and stores 16 bytes: every store
    // instruction writes 4 full 128-byte row segments.
    const int e = warp - kTcEpiWarp0;
    const int q = warp & 3;
    const int h = e >> 2;
    uint8_t* stg = smem + L.stg + (size_t)e * kTcStage;
    const bool out_vec = g.out && ((reinterpret_cast<uintptr_t>(g.out) & 15) == 0) && ((g.ldo & 3) == 0);
    if (g.tma_store && !g.acc) {
      // TMEM -> registers -> dequant (+ReLU) -> 128B-swizzled staging -> one TMA tensor store per
      // 32x32 box (the copy engine writes the rows; ragged rows/columns are clipped by the map).
      int acc = 0;
      uint32_t acc_phase = 0;
      bool pending = false;
      int64_t tile;
      int sl, c0, c1;
      const uint64_t opol = l2_policy(g.out_hint);
      for (int64_t k = 0; item4(k, tile, sl, c0, c1); ++k) {
        mbar_wait(accf_bar + acc, acc_phase);
        tc_fence_after();
        if (warp == kTcEpiWarp0 && lane == 0) stamp(2);
        const int m0 = sl * NS;
        const float* scp = SB ? p.scale + m0 : sc_s;   // scale/offtot of this slice's columns
        const float* otp = SB ? p.offtot + m0 : ot_s;
        const int row0 = (int)(tile * kTcRows) + q * 32;
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * NS);
        for (int j0 = (c0 + ((h - c0) & 1)) * 32; j0 < c1 * 32 && !(g.dbg & 32); j0 += 64) {
          uint32_t v[32];
          tmem_ld16(tbase + j0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
          tmem_ld16(tbase + j0 + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
          tmem_wait_ld();
          float y[32];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 s4 = SB ? __ldg(reinterpret_cast<const float4*>(scp + j0 + 4 * c))
                                 : *reinterpret_cast<const float4*>(scp + j0 + 4 * c);
            const float4 o4 = SB ? __ldg(reinterpret_cast<const float4*>(otp + j0 + 4 * c))
                                 : *reinterpret_cast<const float4*>(otp + j0 + 4 * c);
            y[4 * c + 0] = fmaf(s4.x, u2f_exact(v[4 * c + 0]), o4.x);   // a4, one rounding (R8)
            y[4 * c + 1] = fmaf(s4.y, u2f_exact(v[4 * c + 1]), o4.y);
            y[4 * c + 2] = fmaf(s4.z, u2f_exact(v[4 * c + 2]), o4.z);
            y[4 * c + 3] = fmaf(s4.w, u2f_exact(v[4 * c + 3]), o4.w);
          }
          if (g.relu) {
#pragma unroll
            for (int j = 0; j < 32; ++j) y[j] = relu_pos0(y[j]);
          }
          if (pending) {                              // the previous box has left the staging
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
            if (g.out_hint) tma_store_2d_hint(out_map, stg, m0 + j0, row0, opol);
            else tma_store_2d(out_map, stg, m0 + j0, row0);
            bulk_commit();
          }
          pending = !(g.dbg & 16);
        }
        tc_fence_before();
        mbar_arrive(acce_bar + acc);
        if (warp == kTcEpiWarp0 && lane == 0) stamp(2);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      if (lane == 0) bulk_wait0();
    } else {
    const int cq = lane & 7;                          // 4-column group of this lane in a chunk
    const int rsub = lane >> 3;                       // row within a 4-row store group
    constexpr int kMaxChunks = 4;                     // NS <= 256 -> <= 4 chunks per warp
    float scv[kMaxChunks][4], otv[kMaxChunks][4];
    int cur_sl = -1;
    int acc = 0;
    uint32_t acc_phase = 0;
    int64_t tile;
    int sl, c0, c1;
    for (int64_t k = 0; item4(k, tile, sl, c0, c1); ++k) {
      mbar_wait(accf_bar + acc, acc_phase);
      tc_fence_after();
      const int m0 = sl * NS;
      if (sl != cur_sl) {                             // this lane's scale/offtot, per slice
#pragma unroll
        for (int i = 0; i < kMaxChunks; ++i)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = h * 32 + i * 64 + 4 * cq + u;
            scv[i][u] = j < NS ? (SB ? __ldg(p.scale + m0 + j) : sc_s[j]) : 0.f;
            otv[i][u] = j < NS ? (SB ? __ldg(p.offtot + m0 + j) : ot_s[j]) : 0.f;
          }
        cur_sl = sl;
      }
      const int64_t row0 = tile * kTcRows + q * 32;   // first row of this warp's quadrant
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * NS);
#pragma unroll
      for (int i = 0; i < kMaxChunks; ++i) {
        const int j0 = h * 32 + i * 64;
        if (j0 >= NS) break;
        if (j0 < c0 * 32 || j0 >= c1 * 32) continue;   // outside this item's column range
        uint32_t v[32];
        tmem_ld16(tbase + j0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
        tmem_ld16(tbase + j0 + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
        tmem_wait_ld();
        if (g.acc) {                                  // optional raw int32 output (tests)
          const int64_t row = row0 + lane;
          if (row < g.N) {
            int32_t* a = g.acc + row * g.ldacc + m0 + j0;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (m0 + j0 + j < p.M) a[j] = (int32_t)v[j];
          }
        }
        if (!g.out) continue;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) =
              make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
        __syncwarp();
        const int mcol = m0 + j0 + 4 * cq;
        if (out_vec && row0 + 32 <= g.N && m0 + j0 + 32 <= p.M) {
          // interior chunk: no predicates, one pointer bump per 4 rows
          float* o = g.out + (row0 + rsub) * g.ldo + mcol;
          const int64_t step = 4 * g.ldo;
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int rr = it * 4 + rsub;
            const uint4 a4 = *reinterpret_cast<const uint4*>(stg + rr * 128 + ((cq ^ (rr & 7)) << 4));
            float y0 = fmaf(scv[i][0], u2f_exact(a4.x), otv[i][0]);
            float y1 = fmaf(scv[i][1], u2f_exact(a4.y), otv[i][1]);
            float y2 = fmaf(scv[i][2], u2f_exact(a4.z), otv[i][2]);
            float y3 = fmaf(scv[i][3], u2f_exact(a4.w), otv[i][3]);
            if (g.relu) { y0 = relu_pos0(y0); y1 = relu_pos0(y1); y2 = relu_pos0(y2); y3 = relu_pos0(y3); }
            __stcs(reinterpret_cast<float4*>(o), make_float4(y0, y1, y2, y3));
            o += step;
          }
          __syncwarp();
          continue;
        }
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int rr = it * 4 + rsub;
          const int64_t grow = row0 + rr;
          const uint4 a4 = *reinterpret_cast<const uint4*>(stg + rr * 128 + ((cq ^ (rr & 7)) << 4));
          float y0 = fmaf(scv[i][0], u2f_exact(a4.x), otv[i][0]);
          float y1 = fmaf(scv[i][1], u2f_exact(a4.y), otv[i][1]);
          float y2 = fmaf(scv[i][2], u2f_exact(a4.z), otv[i][2]);
          float y3 = fmaf(scv[i][3], u2f_exact(a4.w), otv[i][3]);
          if (g.relu) { y0 = relu_pos0(y0); y1 = relu_pos0(y1); y2 = relu_pos0(y2); y3 = relu_pos0(y3); }
          if (grow < g.N) {
            float* o = g.out + grow * g.ldo + mcol;
            if (out_vec && mcol + 4 <= p.M) {
              __stcs(reinterpret_cast<float4*>(o), make_float4(y0, y1, y2, y3));
            } else {
              if (mcol + 0 < p.M) o[0] = y0;
              if (mcol + 1 < p.M) o[1] = y1;
              if (mcol + 2 < p.M) o[2] = y2;
              if (mcol + 3 < p.M) o[3] = y3;
            }
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      mbar_arrive(acce_bar + acc);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (span && threadIdx.x == 0) span[1] = gtimer();
  if (warp == kTcMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(g.tmem_cols) : "memory");
  }
}

template <bool FUSED, typename T, bool SB, bool SP = false>
__global__ void __launch_bounds__(kTcThreads, 1) k_tc(DevPlan p, TcKArgs g, const __grid_constant__ CUtensorMap out_map,
                                                      const __grid_constant__ CUtensorMap a_map) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  tc_cta<FUSED, T, SB, SP>(p, g, &out_map, &a_map, smem_raw, blockIdx.x, gridDim.x);
}

// ------------------------------------------------------------------------------ host side
static thread_local const char* g_tc_msg = "";
inline const char* tc_last_msg() { return g_tc_msg; }

// Choose the N slice and build the swizzled K-major LUT image: qt[s][kb][n][128 B] with
// byte (n, k) at sw128_off(n, k/16) + k%16 of block (s, kb); k = 16*(c - 8kb) + code.
inline void tc_layout_host(int C, int M, const uint8_t* lut, TcPlan* t, std::vector<uint8_t>& qt, bool sparse = false) {
  qt.clear();
  t->C = C; t->M = M;
  if (255LL * C >= (1LL << 23)) { t->ok = false; t->why = "C too large for the exact 2^23 float conversion"; return; }
  t->sp = sparse;
  const int ns_hw = sparse ? kSpNsMax : 256;     // TMEM: 2 accumulators (+ sparse metadata) <= 512 columns
  t->KB = (16 * C + kKBlock - 1) / kKBlock;
  int ns_max = (int)(kTcBBudget / ((size_t)t->KB * kKBlock)) / 32 * 32;
  // N per CTA (<= 256).  Note: a 4-slice split of cfg2 (NS = 128) writes its output
  // at 5.36 TB/s, a 4-slice split at 5.84 TB/s (store-pattern probe, profiles/r01).  Developer
  // override (not ABI): ITLUMM_TC_NS_MAX.
  static const int ns_cap = getenv("ITLUMM_TC_NS_MAX") ? atoi(getenv("ITLUMM_TC_NS_MAX")) : 256;
  if (ns_max > ns_cap) ns_max = ns_cap;
  if (ns_max > ns_hw) ns_max = ns_hw;
  // developer override (not ABI): ITLUMM_TC_STREAM=1 streams the LUT even when it could stay resident
  static const bool force_stream = getenv("ITLUMM_TC_STREAM") && atoi(getenv("ITLUMM_TC_STREAM")) != 0;
  // Stream the LUT when it cannot stay resident, and also when residency would force slices
  // narrower than the 256 columns a streamed slice gets (cfg3 C=64: 57.5 us streamed vs 72.8 us
  // resident with 128-column slices; cfg2 C=32 keeps 256-column resident slices: 24.5 vs 31.8 us).
  t->stream_b = ns_max < 32 || force_stream || (ns_max < ns_hw && M > ns_max);
  if (!t->stream_b) {
    // resident slice only if the fused kernel's full layout fits next to it
    const int G0 = (M + ns_max - 1) / ns_max;
    const int NS0 = ((M + G0 - 1) / G0 + 31) / 32 * 32;
    if (tc_smem_layout(C, t->KB, NS0, 1, 16 * ((C + 31) / 32), false, true, kTcStages, sparse).total > kSmemMax)
      t->stream_b = true;
  }
  if (t->stream_b) ns_max = ns_hw;               // LUT K-blocks streamed per stage (large C)
  const int G = (M + ns_max - 1) / ns_max;
  int NS = (M + G - 1) / G;
  NS = (NS + 31) / 32 * 32;                      // whole 32-column epilogue chunks
  t->G = G; t->NS = NS;
  int cols = 32;
  while (cols < 2 * NS) cols <<= 1;
  if (sparse) cols = 512;                        // + 4 metadata columns per ring stage after the accumulators
  t->tmem_cols = cols;
  const size_t blk = (size_t)NS * kKBlock;
  qt.assign((size_t)G * t->KB * blk, 0);
  for (int s = 0; s < G; ++s)
    for (int n = 0; n < NS; ++n) {
      const int m = s * NS + n;
      if (m >= M) continue;
      for (int c = 0; c < C; ++c) {
        const int kb = c / 8, jc = c % 8;
        uint8_t* base = qt.data() + ((size_t)s * t->KB + kb) * blk + sw128_off(n, jc);
        for (int code = 0; code < 16; ++code) base[code] = lut[((size_t)c * 16 + code) * M + m];
      }
    }
  t->ok = true;
  t->why = "";
}

template <bool FUSED, typename T, bool SB, bool SP = false>
inline itlumm_status tc_set_attr(size_t smem) {
  cudaError_t e = cudaFuncSetAttribute((const void*)k_tc<FUSED, T, SB, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) { g_tc_msg = cudaGetErrorString(e); return ITLUMM_ECUDA; }
  return ITLUMM_OK;
}

inline itlumm_status tc_configure(TcPlan& t, int num_sms) {
  if (!t.ok) return ITLUMM_OK;
  // ring depth: 4 stages when they fit next to a 1-stage codes ring, else 3 (developer override,
  // not ABI: ITLUMM_TC_STAGES)
  static const int st_env = getenv("ITLUMM_TC_STAGES") ? atoi(getenv("ITLUMM_TC_STAGES")) : 0;
  t.ST = kTcStages;
  if (st_env >= 2 && st_env <= 6) t.ST = st_env;
  else if (tc_smem_layout(t.C, t.KB, t.NS, 1, 16 * ((t.C + 31) / 32), t.stream_b, !t.stream_b, 4, t.sp).total <= kSmemMax) t.ST = 4;
  if (t.sp && 2 * t.NS + 4 * t.ST > 512) { t.ok = false; t.why = "TMEM budget exceeded (sparse metadata)"; return ITLUMM_OK; }
  t.smem = tc_smem_layout(t.C, t.KB, t.NS, 0, 0, t.stream_b, !t.stream_b, t.ST, t.sp).total;
  if (t.smem > kSmemMax) { t.ok = false; t.why = "shared memory budget exceeded"; return ITLUMM_OK; }
  itlumm_status st;
  if (t.sp) {
    if ((st = tc_set_attr<true, float, false, true>(kSmemMax)) != ITLUMM_OK) return st;
    if ((st = tc_set_attr<true, uint16_t, false, true>(kSmemMax)) != ITLUMM_OK) return st;
    if ((st = tc_set_attr<true, float, true, true>(kSmemMax)) != ITLUMM_OK) return st;
    if ((st = tc_set_attr<true, uint16_t, true, true>(kSmemMax)) != ITLUMM_OK) return st;
    if ((st = tc_set_attr<false, float, false, true>(kSmemMax)) != ITLUMM_OK) return st;
    if ((st = tc_set_attr<false, float, true, true>(kSmemMax)) != ITLUMM_OK) return st;
    t.grid = t.stream_b ? num_sms : t.G * (num_sms / t.G > 0 ? num_sms / t.G : 1);
    return ITLUMM_OK;
  }
  if ((st = tc_set_attr<true, float, false>(kSmemMax)) != ITLUMM_OK) return st;
  if ((st = tc_set_attr<true, uint16_t, false>(kSmemMax)) != ITLUMM_OK) return st;
  if ((st = tc_set_attr<true, float, true>(kSmemMax)) != ITLUMM_OK) return st;
  if ((st = tc_set_attr<true, uint16_t, true>(kSmemMax)) != ITLUMM_OK) return st;
  if ((st = tc_set_attr<false, float, false>(kSmemMax)) != ITLUMM_OK) return st;
  if ((st = tc_set_attr<false, float, true>(kSmemMax)) != ITLUMM_OK) return st;
  t.grid = t.stream_b ? num_sms : t.G * (num_sms / t.G > 0 ? num_sms / t.G : 1);
  return ITLUMM_OK;
}

// AUTO policy: the tensor-core path when its tiling applies.
inline bool tc_preferred(const TcPlan& t, bool simt_ok) { return t.ok || !simt_ok; }

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// Tensor map of `out` (N x M fp32, row stride ldo) with 32x32 boxes and 128-byte swizzle.
inline bool make_out_map(CUtensorMap* map, float* out, int64_t N, int M, int64_t ldo) {
  auto enc = tensor_map_encoder();
  if (!enc || !out || (reinterpret_cast<uintptr_t>(out) & 15) || (ldo & 3) || N < 1 || N > INT32_MAX) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)N};
  const cuuint64_t strides[1] = {(cuuint64_t)ldo * 4};
  const cuuint32_t box[2] = {32, 32};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// `pdl`: launch as a programmatic dependent of the previous kernel on `s` (the encode kernel of
// the TC_PIPE schedule): the prologue overlaps the encode's tail, the codes are read after
// griddepcontrol.wait.
inline itlumm_status tc_launch(const TcPlan& t, const DevPlan& dp, bool fused, bool bf16, const TcArgs& a,
                               cudaStream_t s, bool pdl = false) {
  TcKArgs k{};
  k.A = a.A; k.lda = a.lda; k.codes = a.codes; k.ldc = a.ldc; k.N = a.N;
  k.acc = a.acc; k.ldacc = a.ldacc; k.out = a.out; k.ldo = a.ldo; k.relu = a.relu;
  k.packed = fused && a.packed && (reinterpret_cast<uintptr_t>(a.A) & 15) == 0 &&
             (a.lda * (bf16 ? 2 : 4)) % 16 == 0 ? 1 : 0;
  k.qt = t.qt; k.KB = t.KB; k.NS = t.NS; k.G = t.G; k.tmem_cols = t.tmem_cols;
  k.pdl = pdl ? 1 : 0;
  k.stream_b = t.stream_b ? 1 : 0;
  k.ST = t.ST;
  k.trace = t.trace;
  static const int out_hint = getenv("ITLUMM_OUT_HINT") ? atoi(getenv("ITLUMM_OUT_HINT")) : 0;   // developer
  k.out_hint = out_hint;
  static const int dbg = getenv("ITLUMM_TC_DBG") ? atoi(getenv("ITLUMM_TC_DBG")) : 0;   // developer
  k.dbg = dbg;
  alignas(64) CUtensorMap out_map;
  memset(&out_map, 0, sizeof out_map);
  k.tma_store = (!a.acc && make_out_map(&out_map, a.out, a.N, t.M, a.ldo)) ? 1 : 0;
  // fused over split-packed f32 rows with a resident LUT: rows staged by TMA (developer override,
  // not ABI: ITLUMM_TC_ATMA=0 keeps the per-thread vector loads)
  static const int atma_env = getenv("ITLUMM_TC_ATMA") ? atoi(getenv("ITLUMM_TC_ATMA")) : 1;
  alignas(64) CUtensorMap a_map;
  memset(&a_map, 0, sizeof a_map);
  k.a_tma = 0;
  if (atma_env && k.packed && !bf16 && !t.stream_b && !t.sp && t.C >= 8 && a.N <= INT32_MAX) {
    auto enc = tensor_map_encoder();
    const cuuint64_t dims[2] = {(cuuint64_t)4 * t.C, (cuuint64_t)a.N};
    const cuuint64_t strides[1] = {(cuuint64_t)a.lda * 4};
    const cuuint32_t box[2] = {32, (cuuint32_t)kTcRows};
    const cuuint32_t estr[2] = {1, 1};
    k.a_tma = enc && enc(&a_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(a.A), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS ? 1 : 0;
  }
  size_t smem = t.smem;
  if (fused && t.stream_b) {
    // fused over a streamed LUT: the threshold/column tables sit next to the LUT ring
    smem = tc_smem_layout(t.C, t.KB, t.NS, 0, 0, true, true, t.ST, t.sp).total;
    if (smem > kSmemMax) { g_tc_msg = "fused kernel over a streamed LUT: shared memory budget exceeded"; return ITLUMM_EUNSUPPORTED; }
  }
  k.CS = 0;
  if (!fused && a.ldc % 16 == 0 && (reinterpret_cast<uintptr_t>(a.codes) & 15) == 0) {
    // codes by bulk copy: as many 128-row stages (up to 4) as fit next to the rest (developer
    // override, not ABI: ITLUMM_TC_CS = max codes stages; 0 = producers load codes with __ldg)
    static const int cs_env = getenv("ITLUMM_TC_CS") ? atoi(getenv("ITLUMM_TC_CS")) : 4;
    for (int cs = cs_env; cs >= 1; --cs) {
      const size_t need = tc_smem_layout(t.C, t.KB, t.NS, cs, (int)a.ldc, t.stream_b, fused, t.ST, t.sp).total;
      if (need <= kSmemMax && (int64_t)kTcRows * a.ldc < (1 << 20)) { k.CS = cs; smem = need; break; }
    }
  }
  const int64_t ntiles = (a.N + kTcRows - 1) / kTcRows;
  int64_t grid = t.grid;
  if (grid > (int64_t)t.G * ntiles) grid = (int64_t)t.G * ntiles;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e;
  if (t.sp) {
    if (fused && t.stream_b) e = bf16 ? cudaLaunchKernelEx(&cfg, k_tc<true, uint16_t, true, true>, dp, k, out_map, a_map)
                                      : cudaLaunchKernelEx(&cfg, k_tc<true, float, true, true>, dp, k, out_map, a_map);
    else if (fused) e = bf16 ? cudaLaunchKernelEx(&cfg, k_tc<true, uint16_t, false, true>, dp, k, out_map, a_map)
                             : cudaLaunchKernelEx(&cfg, k_tc<true, float, false, true>, dp, k, out_map, a_map);
    else if (t.stream_b) e = cudaLaunchKernelEx(&cfg, k_tc<false, float, true, true>, dp, k, out_map, a_map);
    else e = cudaLaunchKernelEx(&cfg, k_tc<false, float, false, true>, dp, k, out_map, a_map);
  } else if (fused && t.stream_b) {
    if (bf16) e = cudaLaunchKernelEx(&cfg, k_tc<true, uint16_t, true>, dp, k, out_map, a_map);
    else e = cudaLaunchKernelEx(&cfg, k_tc<true, float, true>, dp, k, out_map, a_map);
  } else if (fused) {
    if (bf16) e = cudaLaunchKernelEx(&cfg, k_tc<true, uint16_t, false>, dp, k, out_map, a_map);
    else e = cudaLaunchKernelEx(&cfg, k_tc<true, float, false>, dp, k, out_map, a_map);
  } else if (t.stream_b) {
    e = cudaLaunchKernelEx(&cfg, k_tc<false, float, true>, dp, k, out_map, a_map);
  } else {
    e = cudaLaunchKernelEx(&cfg, k_tc<false, float, false>, dp, k, out_map, a_map);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) { g_tc_msg = cudaGetErrorString(e); return ITLUMM_ECUDA; }
  return ITLUMM_OK;
}

}  // namespace itlumm
