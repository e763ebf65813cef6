// simt.cuh — CUDA-core kernels of the ITLUMM hot path.
//
//   k_encode          a1+a2: rows -> nibble-packed codes (one thread per output byte).
//   k_lut<MS,FUSED,T> a3+a4: persistent, warp-specialised.  Producer warps turn a tile of R rows
//                     into per-(row, codebook) LUT byte offsets in a shared-memory ring (FUSED:
//                     gather the 4C split columns and walk the trees; else: unpack codes from
//                     HBM).  Consumer warps own MS output columns of the LUT, resident in shared
//                     memory for the whole kernel, and accumulate uint8 entries in 16-bit SWAR
//                     lanes (LDS.128 + PRMT + IMAD), then dequantise (+ReLU) and stream fp32 out.
#pragma once
#include "common.cuh"

namespace itlumm {

// ------------------------------------------------------------------------------- K1 encode
template <typename T>
__global__ void __launch_bounds__(256) k_encode(DevPlan p, const T* __restrict__ A, int64_t lda,
                                                int64_t N, uint8_t* __restrict__ codes,
                                                int64_t ldc) {
  const int nb = (p.C + 1) >> 1;
  const int64_t total = N * nb;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / nb;
    const int b = (int)(idx - r * nb);
    const T* a = A + r * lda;
    float v[2][4];
    const int c0 = 2 * b;
    const bool has1 = (c0 + 1) < p.C;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = has1 ? c0 + h : c0;
      const int4 col = __ldg(reinterpret_cast<const int4*>(p.cols) + c);
      v[h][0] = InTraits<T>::load(a + col.x);
      v[h][1] = InTraits<T>::load(a + col.y);
      v[h][2] = InTraits<T>::load(a + col.z);
      v[h][3] = InTraits<T>::load(a + col.w);
    }
    uint32_t byte = (uint32_t)tree_walk(v[0], p.thr_t, p.C, c0);
    if (has1) byte |= (uint32_t)tree_walk(v[1], p.thr_t, p.C, c0 + 1) << 4;
    codes[r * ldc + b] = (uint8_t)byte;
  }
}

// ------------------------------------------------------------------------------- K3/K4 LUT
constexpr int kProducers = 128;   // 4 producer warps
constexpr int kConsumers = 256;   // 8 consumer warps
constexpr int kLutThreads = kProducers + kConsumers;
constexpr int kMaxStages = 7;     // named barrier ids 1..2*S
constexpr int kPairsPerThread = 8;                        // (row, codebook) pairs per producer chunk
constexpr int kChunkPairs = kProducers * kPairsPerThread; // pairs per producer chunk

struct LutArgs {
  const void* A;          // FUSED: activations
  int64_t lda;
  const uint8_t* codes;   // !FUSED: packed codes
  int64_t ldc;
  int64_t N;
  int32_t* acc;           // optional int32 output
  int64_t ldacc;
  float* out;             // optional fp32 output
  int64_t ldo;
  int relu;
  int vec_out;            // out/acc rows 16-byte aligned -> 128-bit stores
  int R;                  // rows per tile (= rows per consumer pass * RPT)
  int RPT;                // rows per consumer thread per tile
  int S;                  // ring stages
  int G;                  // M slices (grid = G * groups)
  uint32_t one;           // runtime constant 1 (see add_fma_pipe)
};

// Shared-memory footprint (bytes) of k_lut for a plan; mirrors the carve-up in the kernel.
__host__ __device__ inline size_t lut_smem_bytes(int C, int MS, int R, int S, bool fused) {
  const int C4 = (C + 3) & ~3;
  size_t b = (size_t)(C * 16 + 1) * MS;          // LUT slice + one zero row (padding target)
  b = (b + 15) & ~(size_t)15;
  if (fused) b += (size_t)C * 16 + (size_t)15 * C * 4;  // cols [C][4] (16B aligned) + thr [15][C]
  b = (b + 15) & ~(size_t)15;
  b += (size_t)S * R * C4 * 4;                    // offset ring
  return b;
}

// AVG: MADDNESS-style rounded 8-bit summation (reading R22): per group of 16 codebooks a
// 4-level tree of per-byte rounding averages (__vavgu4 on the lane's 16 LUT bytes), group results
// summed exactly; dequant with 16*scale and the bias-corrected offset (DevPlan.offavg).  C % 16 == 0.
template <int MS, bool FUSED, typename T, bool AVG = false>
__global__ void __launch_bounds__(kLutThreads, 1) k_lut(DevPlan p, LutArgs g) {
  constexpr int LPR = MS / 16;               // consumer lanes per row (16 columns each)
  constexpr int RPP = kConsumers / LPR;      // rows per consumer pass
  extern __shared__ __align__(16) uint8_t smem[];
  const int C = p.C;
  const int C4 = (C + 3) & ~3;
  const int R = g.R, S = g.S, G = g.G;
  const int slice = blockIdx.x % G;
  const int group = blockIdx.x / G;
  const int ngroups = gridDim.x / G;
  const int m0 = slice * MS;
  const int64_t ntiles = (g.N + R - 1) / R;

  uint8_t* lut_s = smem;
  size_t off = ((size_t)(C * 16 + 1) * MS + 15) & ~(size_t)15;
  int32_t* cols_s = reinterpret_cast<int32_t*>(smem + off);              // 16-byte aligned
  float* thr_s = reinterpret_cast<float*>(smem + off + (size_t)C * 16);
  if (FUSED) off += (size_t)C * 16 + (size_t)15 * C * 4;
  off = (off + 15) & ~(size_t)15;
  uint32_t* ring = reinterpret_cast<uint32_t*>(smem + off);
  const uint32_t zero_row = (uint32_t)(C * 16 * MS);

  // ---- prologue: LUT slice (columns m0 .. m0+MS) resident for the whole kernel
  {
    const int vec_per_row = MS / 16;
    const int nvec = C * 16 * vec_per_row;
    for (int i = threadIdx.x; i < nvec; i += blockDim.x) {
      const int row = i / vec_per_row, v = i - row * vec_per_row;
      const int m = m0 + v * 16;
      uint4 w = make_uint4(0, 0, 0, 0);
      if (m < p.Mp) w = __ldg(reinterpret_cast<const uint4*>(p.lut + (size_t)row * p.Mp + m));
      reinterpret_cast<uint4*>(lut_s)[i] = w;
    }
    for (int i = threadIdx.x; i < MS / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(lut_s + zero_row)[i] = make_uint4(0, 0, 0, 0);
    if (FUSED) {
      for (int i = threadIdx.x; i < 15 * C; i += blockDim.x) thr_s[i] = __ldg(p.thr_t + i);
      for (int i = threadIdx.x; i < 4 * C; i += blockDim.x) cols_s[i] = __ldg(p.cols + i);
    }
  }
  __syncthreads();

  const int tid = threadIdx.x;
  if (tid < kProducers) {
    // ================================================================ producer warps
    if (FUSED) {
      // The tile sequence is cut into chunks of kChunkPairs (row, codebook) pairs.  The gather
      // of chunk j+1 is issued before the tree walks of chunk j, so the 4 split-column loads of
      // ~2K pairs per CTA are always in flight (latency hiding without occupancy).
      const T* A = reinterpret_cast<const T*>(g.A);
      const int npair = R * C4;
      const int nch = (npair + kChunkPairs - 1) / kChunkPairs;
      float vc[kPairsPerThread][4], vn[kPairsPerThread][4];
      auto load_chunk = [&](int64_t tile, int ch, float (&v)[kPairsPerThread][4]) {
#pragma unroll
        for (int u = 0; u < kPairsPerThread; ++u) {
          const int q = ch * kChunkPairs + u * kProducers + tid;
          const int r = q / C4, c = q - r * C4;
          const int64_t row = tile * R + r;
          if (q < npair && c < C && row < g.N) {
            const int4 col = *reinterpret_cast<const int4*>(cols_s + 4 * c);
            const T* a = A + row * g.lda;
            v[u][0] = InTraits<T>::load(a + col.x);
            v[u][1] = InTraits<T>::load(a + col.y);
            v[u][2] = InTraits<T>::load(a + col.z);
            v[u][3] = InTraits<T>::load(a + col.w);
          }
        }
      };
      int64_t tile = group;
      int ch = 0, k = 0;
      if (tile < ntiles) load_chunk(tile, 0, vc);
      while (tile < ntiles) {
        // next chunk position
        int64_t ntile = tile;
        int nch_i = ch + 1;
        if (nch_i == nch) { nch_i = 0; ntile += ngroups; }
        if (ntile < ntiles) load_chunk(ntile, nch_i, vn);
        const int s = k % S;
        if (ch == 0 && k >= S) named_bar_sync(1 + S + s, kLutThreads);   // stage s released
        uint32_t* st = ring + (size_t)s * R * C4;
#pragma unroll
        for (int u = 0; u < kPairsPerThread; ++u) {
          const int q = ch * kChunkPairs + u * kProducers + tid;
          if (q < npair) {
            const int r = q / C4, c = q - r * C4;
            uint32_t o = zero_row;
            if (c < C && tile * R + r < g.N)
              o = (uint32_t)((c * 16 + tree_walk(vc[u], thr_s, C, c)) * MS);
            st[q] = o;
          }
        }
        if (ch == nch - 1) { named_bar_arrive(1 + s, kLutThreads); ++k; }   // stage s full
#pragma unroll
        for (int u = 0; u < kPairsPerThread; ++u)
#pragma unroll
          for (int t = 0; t < 4; ++t) vc[u][t] = vn[u][t];
        tile = ntile;
        ch = nch_i;
      }
      for (int j = (k > S ? k - S : 0); j < k; ++j) named_bar_sync(1 + S + (j % S), kLutThreads);
    } else {
      int k = 0;
      const int nbp = C4 >> 1;             // byte pairs per row (codebooks 2b, 2b+1)
      const int nb = (C + 1) >> 1;         // real code bytes per row
      const int n = R * nbp;
      for (int64_t tile = group; tile < ntiles; tile += ngroups, ++k) {
        const int s = k % S;
        if (k >= S) named_bar_sync(1 + S + s, kLutThreads);     // consumers released stage s
        uint32_t* st = ring + (size_t)s * R * C4;
        const int64_t row0 = tile * R;
        for (int q = tid; q < n; q += kProducers) {
          const int r = q / nbp, b = q - r * nbp;
          const int64_t row = row0 + r;
          uint32_t o0 = zero_row, o1 = zero_row;
          if (row < g.N && b < nb) {
            const uint32_t byte = g.codes[row * g.ldc + b];
            const int c0 = 2 * b;
            o0 = (uint32_t)((c0 * 16 + (byte & 15)) * MS);
            if (c0 + 1 < C) o1 = (uint32_t)(((c0 + 1) * 16 + (byte >> 4)) * MS);
          }
          *reinterpret_cast<uint2*>(st + r * C4 + 2 * b) = make_uint2(o0, o1);
        }
        named_bar_arrive(1 + s, kLutThreads);                   // stage s full
      }
      for (int j = (k > S ? k - S : 0); j < k; ++j) named_bar_sync(1 + S + (j % S), kLutThreads);
    }
  } else {
    // ================================================================ consumer warps
    const int ctid = tid - kProducers;
    const int rl0 = ctid / LPR;         // first row within the tile
    const int lane = ctid - rl0 * LPR;  // 16-column group within the slice
    const int mbase = m0 + lane * 16;
    float sc[16], ot[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int m = mbase + j;
      sc[j] = (m < p.Mp) ? (AVG ? 16.0f : 1.0f) * __ldg(p.scale + m) : 0.f;   // x16 is exact
      ot[j] = (m < p.Mp) ? __ldg((AVG ? p.offavg : p.offtot) + m) : 0.f;
    }
    const uint32_t one = g.one;
    const bool full = g.vec_out && (mbase + 16 <= p.M);
    int k = 0;
    for (int64_t tile = group; tile < ntiles; tile += ngroups, ++k) {
      const int s = k % S;
      named_bar_sync(1 + s, kLutThreads);
      for (int rr = 0; rr < g.RPT; ++rr) {
        const int rl = rl0 + rr * RPP;
        if (rl >= R) break;
        uint32_t acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0;
        const uint32_t* offs = ring + ((size_t)s * R + rl) * C4;
        const uint8_t* lbase = lut_s + lane * 16;
        if (AVG) {
          for (int g0 = 0; g0 < C4; g0 += 16) {
            uint4 w[16];
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
              const uint4 o = *reinterpret_cast<const uint4*>(offs + g0 + i);
              w[i + 0] = *reinterpret_cast<const uint4*>(lbase + o.x);
              w[i + 1] = *reinterpret_cast<const uint4*>(lbase + o.y);
              w[i + 2] = *reinterpret_cast<const uint4*>(lbase + o.z);
              w[i + 3] = *reinterpret_cast<const uint4*>(lbase + o.w);
            }
#pragma unroll
            for (int n = 16; n > 1; n >>= 1)
#pragma unroll
              for (int i = 0; i < n / 2; ++i) {
                w[i].x = __vavgu4(w[2 * i].x, w[2 * i + 1].x);
                w[i].y = __vavgu4(w[2 * i].y, w[2 * i + 1].y);
                w[i].z = __vavgu4(w[2 * i].z, w[2 * i + 1].z);
                w[i].w = __vavgu4(w[2 * i].w, w[2 * i + 1].w);
              }
            const uint32_t ww[4] = {w[0].x, w[0].y, w[0].z, w[0].w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int b = 0; b < 4; ++b) acc[4 * i + b] += (ww[i] >> (8 * b)) & 0xFFu;
          }
        } else
        for (int cb = 0; cb < C4; cb += 256) {      // 16-bit lanes are exact for <= 257 adds
          uint32_t ev[4] = {0, 0, 0, 0}, od[4] = {0, 0, 0, 0};
          const int ce = min(C4, cb + 256);
#pragma unroll 2
          for (int c = cb; c < ce; c += 4) {
            const uint4 o = *reinterpret_cast<const uint4*>(offs + c);
            const uint4 w0 = *reinterpret_cast<const uint4*>(lbase + o.x);
            const uint4 w1 = *reinterpret_cast<const uint4*>(lbase + o.y);
            const uint4 w2 = *reinterpret_cast<const uint4*>(lbase + o.z);
            const uint4 w3 = *reinterpret_cast<const uint4*>(lbase + o.w);
#define ITLUMM_ACC4(W)                                                             \
  add_fma_pipe(ev[0], even_bytes(W.x), one); add_fma_pipe(od[0], odd_bytes(W.x), one); \
  add_fma_pipe(ev[1], even_bytes(W.y), one); add_fma_pipe(od[1], odd_bytes(W.y), one); \
  add_fma_pipe(ev[2], even_bytes(W.z), one); add_fma_pipe(od[2], odd_bytes(W.z), one); \
  add_fma_pipe(ev[3], even_bytes(W.w), one); add_fma_pipe(od[3], odd_bytes(W.w), one);
            ITLUMM_ACC4(w0) ITLUMM_ACC4(w1) ITLUMM_ACC4(w2) ITLUMM_ACC4(w3)
#undef ITLUMM_ACC4
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {   // word i covers columns 4i..4i+3 of this lane
            acc[4 * i + 0] += ev[i] & 0xFFFFu;
            acc[4 * i + 1] += od[i] & 0xFFFFu;
            acc[4 * i + 2] += ev[i] >> 16;
            acc[4 * i + 3] += od[i] >> 16;
          }
        }
        const int64_t row = tile * R + rl;
        if (row < g.N) {
          if (g.out) {
            float y[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              y[j] = fmaf(sc[j], __uint2float_rn(acc[j]), ot[j]);   // a4, one rounding (R8)
              if (g.relu) y[j] = relu_pos0(y[j]);
            }
            float* o = g.out + row * g.ldo + mbase;
            if (full) {
#pragma unroll
              for (int j = 0; j < 16; j += 4) st_cs_f4(o + j, y[j], y[j + 1], y[j + 2], y[j + 3]);
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (mbase + j < p.M) o[j] = y[j];
            }
          }
          if (g.acc) {
            int32_t* a = g.acc + row * g.ldacc + mbase;
            if (full) {
#pragma unroll
              for (int j = 0; j < 16; j += 4)
                __stcs(reinterpret_cast<int4*>(a + j), make_int4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]));
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (mbase + j < p.M) a[j] = (int32_t)acc[j];
            }
          }
        }
      }
      named_bar_arrive(1 + S + s, kLutThreads);               // stage s free
    }
  }
}

}  // namespace itlumm
