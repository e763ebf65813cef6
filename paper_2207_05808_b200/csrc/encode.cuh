// encode.cuh — a1+a2 streaming encode kernel (SURVEY.md §2.3 K1/K2, B200 form).
//
// Why stream whole rows: the 4C split columns of a row are scattered over it, and DRAM moves whole
// lines, so a gather of 4C values already fetches ~98% of every row (ncu: 3072 of 3136 B per cfg2
// row, profiles/r01).  Reading the rows as one sequential stream through the TMA engine
// (cp.async.bulk -> shared memory, an mbarrier ring of S stages of R rows) reaches full HBM
// bandwidth with one CTA per SM, and the gather then runs from shared memory.
//
// Per persistent CTA: thread 0 keeps S row tiles in flight; every thread waits on the stage's
// mbarrier, gathers the 4 split values of (row, codebook) pairs from shared memory, walks the
// depth-4 trees (thresholds resident in shared memory) and writes nibble-packed code bytes
// (R14) with coalesced stores.  After the tile, a CTA barrier frees the stage and thread 0
// refills it with the tile S steps ahead.
#pragma once
#include "common.cuh"

namespace itlumm {

constexpr int kEncConsumerWarps = 16;                         // default consumer warps
constexpr int kEncMaxConsumerWarps = 24;

struct EncArgs {
  const void* A;
  int64_t lda;          // elements
  int64_t N;
  uint8_t* codes;
  int64_t ldc;
  int R;                // rows per stage
  int S;                // stages
  int row_bytes;        // bytes of one staged row (D * es, multiple of 16)
  int contiguous;       // lda == D: a tile is one bulk copy
  int pdl;              // let a dependent grid launch early (PDL)
  int fixed_ok;         // developer switch for the register-threshold WIDE consumer (1 = allowed)
  int packed;           // split-packed rows: cols[c][t] == 4c + t (one vector load per codebook)
  int pdl_wait;         // launched as a programmatic dependent: wait for the previous grid before reading A
  int a_hint;           // L2 policy of the row reads (l2_policy kind; 0 = default)
  uint64_t* span;       // developer trace: [cta][2] globaltimer at CTA start / end (or null)
};

// Shared-memory footprint: [S][R][row_bytes] rows | cols [C][4] | thr [15][C] | 2S mbarriers.
__host__ __device__ inline size_t enc_smem_bytes(int C, int R, int S, int row_bytes) {
  size_t o = (size_t)S * R * row_bytes;
  o += (size_t)15 * C * 4 + (size_t)C * 16;
  o = (o + 15) & ~(size_t)15;
  o += (size_t)2 * S * 8;
  return o;
}

// Warp 0 lane 0 keeps S row tiles in flight (full[s]: bytes landed; empty[s]: every consumer warp
// is done with the stage).  Consumer warps take (row, 32-codebook group) units of a tile: lane l
// walks the tree of codebook 32u+l, adjacent lanes pair their nibbles with one shuffle and the
// even lane stores the byte.  No CTA-wide barrier in the loop: warps drift across stages freely.
// One persistent encoder CTA (`cta` of `ncta`) with warp 0 as the bulk-copy producer and
// blockDim/32 - 1 consumer warps.
// WIDE (C >= 32): a warp unit is one 32-codebook group of one row, units taken in turn; the
// general (row, codebook) lane mapping below is compiled out (it measured slower for C = 256:
// cfg4 layer-1 encode 685 -> 783 us, when both lived in one kernel).
template <typename T, bool WIDE>
__device__ __forceinline__ void enc_cta(const DevPlan& p, const EncArgs& g, uint8_t* smem, int cta, int ncta) {
  const int nconsumer = (int)(blockDim.x >> 5) - 1;
  const int C = p.C, R = g.R, S = g.S, rb = g.row_bytes;
  const int rs = rb / (int)sizeof(T);                 // staged row stride (elements)
  uint8_t* rows_s = smem;
  int32_t* cols_s = reinterpret_cast<int32_t*>(smem + (size_t)S * R * rb);   // 16-byte aligned
  float* thr_s = reinterpret_cast<float*>(cols_s + 4 * C);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (((size_t)S * R * rb + (size_t)15 * C * 4 + (size_t)C * 16 + 15) & ~(size_t)15));
  uint64_t* empty = full + S;
  const int64_t ntiles = (g.N + R - 1) / R;
  const char* A = reinterpret_cast<const char*>(g.A);
  const size_t ldab = (size_t)g.lda * sizeof(T);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (g.span && threadIdx.x == 0) g.span[2 * cta] = gtimer_ns();

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, nconsumer); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 15 * C; i += blockDim.x) thr_s[i] = __ldg(p.thr_t + i);
  for (int i = threadIdx.x; i < 4 * C; i += blockDim.x) cols_s[i] = __ldg(p.cols + i);
  __syncthreads();
  if (g.pdl_wait) pdl_wait();         // A and the codes buffer belong to the stream order
  if (g.pdl) pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      int k = 0;
      const uint64_t pol = l2_policy(g.a_hint);
      for (int64_t tile = cta; tile < ntiles; tile += ncta, ++k) {
        const int s = k % S;
        if (k >= S) mbar_wait(empty + s, (uint32_t)(((k / S) - 1) & 1));
        const int64_t r0 = tile * R;
        const int rows = (int)((g.N - r0) < R ? (g.N - r0) : R);
        uint8_t* dst = rows_s + (size_t)s * R * rb;
        mbar_arrive_expect_tx(full + s, (uint32_t)rows * rb);
        if (g.contiguous) {
          if (g.a_hint) bulk_g2s_hint(dst, A + r0 * ldab, (uint32_t)rows * rb, full + s, pol);
          else bulk_g2s(dst, A + r0 * ldab, (uint32_t)rows * rb, full + s);
        } else {
          for (int r = 0; r < rows; ++r) bulk_g2s(dst + (size_t)r * rb, A + (r0 + r) * ldab, rb, full + s);
        }
      }
    }
    return;
  }
  const int cw = warp - 1;
  // lanes per row: the codebooks of a row (rounded up to a power of two, >= 2 so that adjacent
  // lanes pair their nibbles, <= 32); a warp unit covers 32 / lpr rows (short rows, small C) or one
  // 32-codebook group of one row (C > 32)
  int lpr = 2;
  while (lpr < C && lpr < 32) lpr <<= 1;
  const int rpu = 32 / lpr;                            // rows per warp unit
  const int ngrp = (C + 31) >> 5;                      // 32-codebook groups per row
  const int rsub = lane / lpr, cl = lane - rsub * lpr;
  // WIDE with 32-codebook groups that divide the consumer warps (C = 32, 64, 128, 256): warp cw
  // always serves group cw % ngrp, so each lane owns one codebook for the whole kernel and keeps
  // its 15 thresholds and 4 gather columns in registers; the tree walk is then compare/select only
  // (no dependent shared-memory loads), and two rows are walked per pass for ILP.
  const bool fixed = WIDE && (nconsumer % ngrp) == 0 && g.fixed_ok;
  const int fc = (cw % ngrp) * 32 + lane;              // this lane's codebook (fixed mode)
  float tr[15];
  int4 fcol = make_int4(0, 0, 0, 0);
  if (fixed && fc < C) {
#pragma unroll
    for (int h = 0; h < 15; ++h) tr[h] = thr_s[h * C + fc];
    fcol = *reinterpret_cast<const int4*>(cols_s + 4 * fc);
  } else {
#pragma unroll
    for (int h = 0; h < 15; ++h) tr[h] = 0.f;
  }
  auto walk_regs = [&](float v0, float v1, float v2, float v3) -> uint32_t {
    const uint32_t b0 = v0 > tr[0];
    const uint32_t b1 = v1 > (b0 ? tr[2] : tr[1]);
    const float t2a = b1 ? tr[4] : tr[3], t2b = b1 ? tr[6] : tr[5];
    const uint32_t b2 = v2 > (b0 ? t2b : t2a);
    const float x0 = b2 ? tr[8] : tr[7], x1 = b2 ? tr[10] : tr[9], x2 = b2 ? tr[12] : tr[11], x3 = b2 ? tr[14] : tr[13];
    const float y0 = b1 ? x1 : x0, y1 = b1 ? x3 : x2;
    const uint32_t b3 = v3 > (b0 ? y1 : y0);
    return (b0 << 3) | (b1 << 2) | (b2 << 1) | b3;
  };
  auto load4 = [&](const T* a, float& v0, float& v1, float& v2, float& v3) {
    if (g.packed) {
      if (sizeof(T) == 4) {
        const float4 q = *reinterpret_cast<const float4*>(a + 4 * fc);
        v0 = q.x; v1 = q.y; v2 = q.z; v3 = q.w;
      } else {
        const uint2 q = *reinterpret_cast<const uint2*>(a + 4 * fc);
        v0 = __uint_as_float(q.x << 16); v1 = __uint_as_float(q.x & 0xFFFF0000u);
        v2 = __uint_as_float(q.y << 16); v3 = __uint_as_float(q.y & 0xFFFF0000u);
      }
    } else {
      v0 = InTraits<T>::lds(a + fcol.x); v1 = InTraits<T>::lds(a + fcol.y);
      v2 = InTraits<T>::lds(a + fcol.z); v3 = InTraits<T>::lds(a + fcol.w);
    }
  };
  int k = 0;
  for (int64_t tile = cta; tile < ntiles; tile += ncta, ++k) {
    const int s = k % S;
    mbar_wait(full + s, (uint32_t)((k / S) & 1));
    const T* rows = reinterpret_cast<const T*>(rows_s + (size_t)s * R * rb);
    const int64_t r0 = tile * R;
    const int nrows = (int)((g.N - r0) < R ? (g.N - r0) : R);
    const int nunits = ((nrows + rpu - 1) / rpu) * ngrp;
    if (WIDE && fixed) {
      const int rstep = nconsumer / ngrp;
      const bool valid = fc < C;
      for (int r = cw / ngrp; r < nrows; r += 2 * rstep) {
        const int r2 = r + rstep;
        uint32_t code = 0, code2 = 0;
        if (valid) {
          float v0, v1, v2, v3, w0, w1, w2, w3;
          load4(rows + (size_t)r * rs, v0, v1, v2, v3);
          if (r2 < nrows) load4(rows + (size_t)r2 * rs, w0, w1, w2, w3);
          else w0 = w1 = w2 = w3 = 0.f;
          code = walk_regs(v0, v1, v2, v3);
          code2 = walk_regs(w0, w1, w2, w3);
        }
        const uint32_t hi = __shfl_down_sync(0xffffffffu, code, 1);
        const uint32_t hi2 = __shfl_down_sync(0xffffffffu, code2, 1);
        if (!(lane & 1) && valid) {
          g.codes[(r0 + r) * g.ldc + (fc >> 1)] = (uint8_t)(code | (hi << 4));
          if (r2 < nrows) g.codes[(r0 + r2) * g.ldc + (fc >> 1)] = (uint8_t)(code2 | (hi2 << 4));
        }
      }
    } else if (WIDE) {
      for (int u = cw; u < nrows * ngrp; u += nconsumer) {
        const int r = u / ngrp, grp = u - r * ngrp;
        const int c = grp * 32 + lane;
        uint32_t code = 0;
        if (c < C) {
          const T* a = rows + (size_t)r * rs;
          const int4 col = *reinterpret_cast<const int4*>(cols_s + 4 * c);
          float v[4];
          v[0] = InTraits<T>::lds(a + col.x);
          v[1] = InTraits<T>::lds(a + col.y);
          v[2] = InTraits<T>::lds(a + col.z);
          v[3] = InTraits<T>::lds(a + col.w);
          code = (uint32_t)tree_walk(v, thr_s, C, c);
        }
        const uint32_t hi = __shfl_down_sync(0xffffffffu, code, 1);
        if (!(lane & 1) && c < C) g.codes[(r0 + r) * g.ldc + (c >> 1)] = (uint8_t)(code | (hi << 4));
      }
    } else if (nunits <= nconsumer) {                         // at most one unit per warp (cfg2 shapes)
      if (cw < nunits) {
        const int ur = cw / ngrp, grp = cw - ur * ngrp;
        const int r = ur * rpu + rsub, c = grp * 32 + cl;
        uint32_t code = 0;
        if (r < nrows && c < C) {
          const T* a = rows + (size_t)r * rs;
          const int4 col = *reinterpret_cast<const int4*>(cols_s + 4 * c);
          float v[4];
          v[0] = InTraits<T>::lds(a + col.x);
          v[1] = InTraits<T>::lds(a + col.y);
          v[2] = InTraits<T>::lds(a + col.z);
          v[3] = InTraits<T>::lds(a + col.w);
          code = (uint32_t)tree_walk(v, thr_s, C, c);
        }
        const uint32_t hi = __shfl_down_sync(0xffffffffu, code, 1);
        if (!(lane & 1) && r < nrows && c < C) g.codes[(r0 + r) * g.ldc + (c >> 1)] = (uint8_t)(code | (hi << 4));
      }
    } else
    // short rows (C < 32): two units per pass, their shared-memory gathers and tree walks overlap
    for (int u0 = cw; u0 < nunits; u0 += 2 * nconsumer) {
      uint32_t code[2];
      int rr[2], cc[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = u0 + h * nconsumer;
        const int ur = u / ngrp, grp = u - ur * ngrp;
        rr[h] = ur * rpu + rsub;
        cc[h] = grp * 32 + cl;
        code[h] = 0;
        if (u < nunits && rr[h] < nrows && cc[h] < C) {
          const T* a = rows + (size_t)rr[h] * rs;
          const int4 col = *reinterpret_cast<const int4*>(cols_s + 4 * cc[h]);
          float v[4];
          v[0] = InTraits<T>::lds(a + col.x);
          v[1] = InTraits<T>::lds(a + col.y);
          v[2] = InTraits<T>::lds(a + col.z);
          v[3] = InTraits<T>::lds(a + col.w);
          code[h] = (uint32_t)tree_walk(v, thr_s, C, cc[h]);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = u0 + h * nconsumer;
        const uint32_t hi = __shfl_down_sync(0xffffffffu, code[h], 1);
        if (u < nunits && !(lane & 1) && rr[h] < nrows && cc[h] < C)
          g.codes[(r0 + rr[h]) * g.ldc + (cc[h] >> 1)] = (uint8_t)(code[h] | (hi << 4));
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);             // releases this warp's code stores (CTA scope)
  }
  if (g.span && cw == 0 && lane == 0) g.span[2 * cta + 1] = gtimer_ns();
}

template <typename T, bool WIDE>
__global__ void __launch_bounds__(32 * (1 + kEncMaxConsumerWarps), 1) k_encode_rows(DevPlan p, EncArgs g) {
  extern __shared__ __align__(16) uint8_t smem_enc[];
  enc_cta<T, WIDE>(p, g, smem_enc, blockIdx.x, gridDim.x);
}

}  // namespace itlumm
