// itlumm.cu — host library behind include/itlumm.h: plan validation, permutation folding,
// parameter layout on the device, kernel selection and launches, the pipelined host API.
// Every arithmetic step of the hot path runs in the kernels (simt.cuh, tc.cuh); the host only
// validates, re-lays-out parameters once per plan, and launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/itlumm.h"
#include "common.cuh"
#include "encode.cuh"
#include "simt.cuh"
#include "tc.cuh"
#include "tcp.cuh"

using namespace itlumm;

// ------------------------------------------------------------------------------ errors
static thread_local std::string g_err;
static thread_local int32_t g_launches = 0;

static itlumm_status fail(itlumm_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess) return fail(ITLUMM_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

// ------------------------------------------------------------------------------ plan
struct SimtCfg {
  int MS = 0, R = 0, S = 0, G = 0, RPT = 1;
  size_t smem_fused = 0, smem_codes = 0;
  int grid_fused = 0, grid_codes = 0;
};

struct itlumm_plan_s {
  int device = 0;
  int D = 0, C = 0, M = 0, Mp = 0;
  int num_sms = 0;
  itlumm_algo algo = ITLUMM_ALGO_AUTO;
  itlumm_summation summation = ITLUMM_SUM_EXACT;
  void* dmem = nullptr;  // one allocation holding every device parameter
  DevPlan dp{};
  SimtCfg simt{};
  TcPlan tc{};
  TcPlan tcs{};                  // the same tiling with the 2:4-sparse one-hot (f2)
  itlumm_onehot onehot = ITLUMM_ONEHOT_AUTO;
  TcpPlan pair_sp{};             // CTA-pair kernel over the sparse tiling (streamed LUT), AUTO's choice
  TcpPlan pair_dn{};             // the same over the dense tiling
  // TC_PIPE code scratch (allocated at plan creation; reuse ordered by scratch_ev)
  std::mutex scratch_mu;
  uint8_t* scratch = nullptr;
  int64_t scratch_rows = 0, scratch_ldc = 0;
  cudaEvent_t scratch_ev = nullptr;
  bool scratch_used = false;
  double seg_frac[2] = {1.0, 1.0};  // fraction of a row's 64-byte segments the gather touches (f32, bf16)
  bool packed = false;           // split-packed input: gather column of (c, t) is 4c + t
  // host API staging
  std::mutex host_mu;
  cudaStream_t hs[3] = {nullptr, nullptr, nullptr};   // host API: 3-stage copy/compute ring
  cudaEvent_t hev = nullptr;
  void* stage = nullptr;
  size_t stage_bytes = 0;
};

static bool finite_all(const float* v, int n) {
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

typedef void (*lut_kernel_t)(DevPlan, LutArgs);

template <bool FUSED, typename T, bool AVG = false>
static lut_kernel_t pick_lut_kernel(int MS) {
  switch (MS) {
    case 16: return k_lut<16, FUSED, T, AVG>;
    case 32: return k_lut<32, FUSED, T, AVG>;
    case 64: return k_lut<64, FUSED, T, AVG>;
    case 128: return k_lut<128, FUSED, T, AVG>;
    case 256: return k_lut<256, FUSED, T, AVG>;
  }
  return nullptr;
}

static itlumm_status set_smem(lut_kernel_t k, size_t smem) {
  CUDA_TRY(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return ITLUMM_OK;
}

// Choose the SIMT tiling: the widest power-of-two M slice whose LUT stays resident in shared
// memory, then the tile height and ring depth.
static itlumm_status configure_simt(itlumm_plan_s* P) {
  const int C = P->C;
  const size_t budget = 200 * 1024;
  int mp2 = 16;
  while (mp2 < P->Mp && mp2 < 256) mp2 <<= 1;
  const int C4 = (C + 3) & ~3;
  for (int MS = mp2; MS >= 16; MS >>= 1) {
    const int LPR = MS / 16;
    const int RPP = kConsumers / LPR;
    // rows per tile: grow by whole consumer passes until a tile holds >= one producer chunk
    // of (row, codebook) pairs, keeping the offset ring <= 48 KB
    int RPT = 1;
    while (RPT < 8 && (int64_t)RPP * RPT * C4 < kChunkPairs) RPT <<= 1;
    int R = RPP * RPT;
    int S = 4;
    while (R > 1 && (size_t)S * R * C4 * 4 > 48 * 1024) {
      if (RPT > 1) RPT >>= 1;
      R >>= 1;
    }
    if (lut_smem_bytes(C, MS, R, S, true) <= budget) {
      SimtCfg& s = P->simt;
      s.MS = MS; s.R = R; s.S = S; s.RPT = RPT;
      s.G = (P->Mp + MS - 1) / MS;
      s.smem_fused = lut_smem_bytes(C, MS, R, S, true);
      s.smem_codes = lut_smem_bytes(C, MS, R, S, false);
      lut_kernel_t kf32 = pick_lut_kernel<true, float>(MS), kbf = pick_lut_kernel<true, uint16_t>(MS),
                   kc = pick_lut_kernel<false, float>(MS);
      itlumm_status st;
      if ((st = set_smem(kf32, s.smem_fused)) != ITLUMM_OK) return st;
      if ((st = set_smem(kbf, s.smem_fused)) != ITLUMM_OK) return st;
      if ((st = set_smem(kc, s.smem_codes)) != ITLUMM_OK) return st;
      if ((st = set_smem(pick_lut_kernel<true, float, true>(MS), s.smem_fused)) != ITLUMM_OK) return st;
      if ((st = set_smem(pick_lut_kernel<true, uint16_t, true>(MS), s.smem_fused)) != ITLUMM_OK) return st;
      if ((st = set_smem(pick_lut_kernel<false, float, true>(MS), s.smem_codes)) != ITLUMM_OK) return st;
      int occ_f = 0, occ_c = 0;
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_f, kf32, kLutThreads, s.smem_fused));
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_c, kc, kLutThreads, s.smem_codes));
      occ_f = std::max(occ_f, 1);
      occ_c = std::max(occ_c, 1);
      s.grid_fused = s.G * std::max(1, P->num_sms * occ_f / s.G);
      s.grid_codes = s.G * std::max(1, P->num_sms * occ_c / s.G);
      return ITLUMM_OK;
    }
  }
  return ITLUMM_OK;  // simt.MS == 0: SIMT kernels unsupported for this C (C > ~780)
}

// Column views used when layers are chained (itlumm_mlp): out_cols selects and orders the output
// columns the plan computes (the only ones the next layer reads); in_map relocates the logical
// input dims into a compacted input row of width D_in (the previous layer's selected columns).
struct PlanView {
  const int32_t* out_cols = nullptr;
  int n_out = 0;
  const int32_t* in_map = nullptr;   // [D] -> column in [0, D_in) or -1 (never a split column)
  int D_in = 0;
};

static itlumm_status plan_create_impl(const itlumm_params* p0, int cuda_device, const PlanView& v,
                                      itlumm_plan* out) {
  g_err.clear();
  if (!out) return fail(ITLUMM_EINVAL, "out is NULL");
  *out = nullptr;
  if (!p0) return fail(ITLUMM_EINVAL, "params is NULL");
  // output column selection: a params copy pointing at the selected LUT columns
  itlumm_params sel = *p0;
  std::vector<uint8_t> lut_sel;
  std::vector<float> sc_sel, off_sel, bias_sel;
  if (v.out_cols) {
    if (v.n_out < 1 || !p0->lut || !p0->scale || !p0->offset) return fail(ITLUMM_EINVAL, "bad output column selection");
    const int Mf = p0->M, Ms = v.n_out;
    lut_sel.resize((size_t)p0->C * 16 * Ms);
    sc_sel.resize(Ms); off_sel.resize(Ms); bias_sel.resize(Ms);
    for (int j = 0; j < Ms; ++j) {
      const int m = v.out_cols[j];
      if (m < 0 || m >= Mf) return fail(ITLUMM_EINVAL, "output column %d outside [0, %d)", m, Mf);
      sc_sel[j] = p0->scale[m]; off_sel[j] = p0->offset[m]; bias_sel[j] = p0->bias ? p0->bias[m] : 0.f;
      for (size_t r = 0; r < (size_t)p0->C * 16; ++r) lut_sel[r * Ms + j] = p0->lut[r * Mf + m];
    }
    sel.M = Ms; sel.lut = lut_sel.data(); sel.scale = sc_sel.data(); sel.offset = off_sel.data(); sel.bias = bias_sel.data();
  }
  const itlumm_params* p = &sel;
  const int D = p->D, C = p->C, M = p->M;
  if (D < 1 || C < 1 || M < 1) return fail(ITLUMM_EINVAL, "D, C, M must be >= 1 (got %d, %d, %d)", D, C, M);
  if (C > D) return fail(ITLUMM_EINVAL, "C (%d) > D (%d)", C, D);
  if (!p->split_dim || !p->thresholds || !p->lut || !p->scale || !p->offset)
    return fail(ITLUMM_EINVAL, "split_dim, thresholds, lut, scale and offset are required");
  // a1: permutation and partition
  std::vector<int32_t> perm(D), bnd(C + 1);
  if (p->perm) {
    std::vector<char> seen(D, 0);
    for (int i = 0; i < D; ++i) {
      const int v = p->perm[i];
      if (v < 0 || v >= D || seen[v]) return fail(ITLUMM_EINVAL, "perm is not a bijection of [0, D) (perm[%d] = %d)", i, v);
      seen[v] = 1;
      perm[i] = v;
    }
  } else {
    for (int i = 0; i < D; ++i) perm[i] = i;
  }
  if (p->boundaries) {
    for (int c = 0; c <= C; ++c) bnd[c] = p->boundaries[c];
    if (bnd[0] != 0 || bnd[C] != D) return fail(ITLUMM_EINVAL, "boundaries must start at 0 and end at D");
    for (int c = 0; c < C; ++c)
      if (bnd[c + 1] <= bnd[c]) return fail(ITLUMM_EINVAL, "boundaries not strictly increasing at %d", c);
  } else {
    const int q = D / C, r = D % C;  // reading R12: larger chunks first
    bnd[0] = 0;
    for (int c = 0; c < C; ++c) bnd[c + 1] = bnd[c] + q + (c < r ? 1 : 0);
  }
  std::vector<int32_t> cols(4 * (size_t)C);
  for (int c = 0; c < C; ++c)
    for (int t = 0; t < kLevels; ++t) {
      const int sd = p->split_dim[c * 4 + t];
      if (sd < 0 || sd >= bnd[c + 1] - bnd[c])
        return fail(ITLUMM_EINVAL, "split_dim[%d][%d] = %d outside [0, %d)", c, t, sd, bnd[c + 1] - bnd[c]);
      cols[c * 4 + t] = perm[bnd[c] + sd];   // folded gather column
    }
  if (v.in_map) {                              // compacted input row (chained layer)
    if (v.D_in < 1) return fail(ITLUMM_EINVAL, "bad input width");
    for (auto& col : cols) {
      const int m = v.in_map[col];
      if (m < 0 || m >= v.D_in) return fail(ITLUMM_EINVAL, "split column %d missing from the compacted input", col);
      col = m;
    }
  }
  for (int i = 0; i < C * 15; ++i)
    if (std::isnan(p->thresholds[i])) return fail(ITLUMM_EINVAL, "threshold %d is NaN", i);
  if (!finite_all(p->scale, M) || !finite_all(p->offset, M) || (p->bias && !finite_all(p->bias, M)))
    return fail(ITLUMM_EINVAL, "scale/offset/bias must be finite");

  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (cuda_device < 0 || cuda_device >= ndev) return fail(ITLUMM_EINVAL, "bad cuda_device %d (have %d)", cuda_device, ndev);

  itlumm_plan_s* P = new (std::nothrow) itlumm_plan_s();
  if (!P) return fail(ITLUMM_ENOMEM, "host allocation failed");
  P->device = cuda_device;
  P->D = v.in_map ? v.D_in : D; P->C = C; P->M = M; P->Mp = (M + 15) & ~15;
  for (int d = 0; d < 2; ++d) {               // DRAM lines a per-column gather of a row touches
    const int es = d == 0 ? 4 : 2;
    const int nseg = (P->D * es + 63) / 64;
    std::vector<char> hit(nseg, 0);
    int n = 0;
    for (int col : cols) { const int sgi = col * es / 64; if (!hit[sgi]) { hit[sgi] = 1; ++n; } }
    P->seg_frac[d] = (double)n / nseg;
  }
  P->packed = true;
  for (int i = 0; i < 4 * C; ++i) P->packed = P->packed && cols[i] == i;
  const int Mp = P->Mp;

  // host images of the device parameters
  std::vector<float> thr_t((size_t)15 * C);
  for (int c = 0; c < C; ++c)
    for (int h = 0; h < 15; ++h) thr_t[(size_t)h * C + c] = p->thresholds[c * 15 + h];
  std::vector<uint8_t> lut((size_t)C * 16 * Mp, 0);
  for (size_t r = 0; r < (size_t)C * 16; ++r) memcpy(&lut[r * Mp], p->lut + r * M, M);
  std::vector<uint8_t> qt, qs;
  tc_layout_host(C, M, p->lut, &P->tc, qt);
  tc_layout_host(C, M, p->lut, &P->tcs, qs, true);
  const int Mpad = std::max({Mp, P->tc.ok ? P->tc.G * P->tc.NS : 0, P->tcs.ok ? P->tcs.G * P->tcs.NS : 0});   // slice columns past M read 0
  std::vector<float> scale(Mpad, 0.f), offtot(Mpad, 0.f), offavg(Mpad, 0.f);
  for (int m = 0; m < M; ++m) {
    scale[m] = p->scale[m];
    const double b = p->bias ? (double)p->bias[m] : 0.0;
    offtot[m] = (float)((double)C * (double)p->offset[m] + b);   // reading R8
    // avg16 summation (reading R22): the rounding-average tree over-estimates each group mean by
    // +1 in expectation; 16 * (C/16) * scale removes it
    offavg[m] = (float)((double)C * (double)p->offset[m] + b - 16.0 * (C / 16) * (double)p->scale[m]);
  }

  // one device allocation
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t o_cols = 0, o_thr = o_cols + al(cols.size() * 4), o_lut = o_thr + al(thr_t.size() * 4),
               o_sc = o_lut + al(lut.size()), o_ot = o_sc + al((size_t)Mpad * 4), o_oa = o_ot + al((size_t)Mpad * 4),
               o_qt = o_oa + al((size_t)Mpad * 4), o_qs = o_qt + al(qt.size()),
               total = o_qs + al(qs.size());
  int prev = 0;
  cudaGetDevice(&prev);
  auto cleanup = [&](itlumm_status st) {
    if (P->dmem) cudaFree(P->dmem);
    if (P->scratch) cudaFree(P->scratch);
    if (P->scratch_ev) cudaEventDestroy(P->scratch_ev);
    delete P;
    cudaSetDevice(prev);
    return st;
  };
  cudaError_t e = cudaSetDevice(cuda_device);
  if (e != cudaSuccess) return cleanup(fail(ITLUMM_ECUDA, "cudaSetDevice: %s", cudaGetErrorString(e)));
  cudaDeviceGetAttribute(&P->num_sms, cudaDevAttrMultiProcessorCount, cuda_device);
  e = cudaMalloc(&P->dmem, total);
  if (e != cudaSuccess) return cleanup(fail(ITLUMM_ENOMEM, "cudaMalloc(%zu): %s", total, cudaGetErrorString(e)));
  uint8_t* base = (uint8_t*)P->dmem;
  struct { size_t off; const void* src; size_t n; } cp[] = {
      {o_cols, cols.data(), cols.size() * 4}, {o_thr, thr_t.data(), thr_t.size() * 4},
      {o_lut, lut.data(), lut.size()},        {o_sc, scale.data(), (size_t)Mpad * 4},
      {o_ot, offtot.data(), (size_t)Mpad * 4},  {o_oa, offavg.data(), (size_t)Mpad * 4},
      {o_qt, qt.data(), qt.size()},           {o_qs, qs.data(), qs.size()}};
  for (auto& c : cp) {
    if (!c.n) continue;
    e = cudaMemcpy(base + c.off, c.src, c.n, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cleanup(fail(ITLUMM_ECUDA, "cudaMemcpy: %s", cudaGetErrorString(e)));
  }
  P->dp.cols = (const int32_t*)(base + o_cols);
  P->dp.thr_t = (const float*)(base + o_thr);
  P->dp.lut = base + o_lut;
  P->dp.scale = (const float*)(base + o_sc);
  P->dp.offtot = (const float*)(base + o_ot);
  P->dp.offavg = (const float*)(base + o_oa);
  P->dp.D = P->D; P->dp.C = C; P->dp.M = M; P->dp.Mp = Mp;
  P->tc.qt = qt.empty() ? nullptr : base + o_qt;
  P->tcs.qt = qs.empty() ? nullptr : base + o_qs;
  cudaFuncSetAttribute((const void*)k_encode_rows<float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute((const void*)k_encode_rows<uint16_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute((const void*)k_encode_rows<float, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute((const void*)k_encode_rows<uint16_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  itlumm_status st = configure_simt(P);
  if (st != ITLUMM_OK) return cleanup(st);
  st = tc_configure(P->tc, P->num_sms);
  if (st == ITLUMM_OK) st = tc_configure(P->tcs, P->num_sms);
  if (st == ITLUMM_OK && getenv("ITLUMM_TC_TRACE") && atoi(getenv("ITLUMM_TC_TRACE")) != 0) {
    cudaMalloc(&P->tc.trace, ((size_t)16 * 4 * kTraceEv + 4 * 512) * 8);
    if (P->tc.trace) cudaMemset(P->tc.trace, 0, ((size_t)16 * 4 * kTraceEv + 4 * 512) * 8);
    P->tcs.trace = P->tc.trace;
  }
  if (st != ITLUMM_OK) return cleanup(fail(st, "%s", tc_last_msg()));
  if (P->tcs.ok && P->tcs.stream_b) tcp_configure(P->pair_sp, P->tcs, P->num_sms);
  if (P->tc.ok && P->tc.stream_b) tcp_configure(P->pair_dn, P->tc, P->num_sms);
  P->pair_sp.trace = P->pair_dn.trace = P->tc.trace;
  if (P->tc.ok || P->tcs.ok) {
    P->scratch_ldc = (((C + 1) / 2) + 15) & ~15;
    P->scratch_rows = 262144;
    e = cudaMalloc(&P->scratch, (size_t)P->scratch_rows * P->scratch_ldc);
    if (e != cudaSuccess) return cleanup(fail(ITLUMM_ENOMEM, "scratch cudaMalloc: %s", cudaGetErrorString(e)));
    e = cudaEventCreateWithFlags(&P->scratch_ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return cleanup(fail(ITLUMM_ECUDA, "cudaEventCreate: %s", cudaGetErrorString(e)));
  }
  cudaSetDevice(prev);
  *out = P;
  return ITLUMM_OK;
}

extern "C" itlumm_status itlumm_plan_create(const itlumm_params* p, int cuda_device, itlumm_plan* out) {
  return plan_create_impl(p, cuda_device, PlanView{}, out);
}

extern "C" itlumm_status itlumm_plan_destroy(itlumm_plan P) {
  g_err.clear();
  if (!P) return ITLUMM_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(P->device);
  cudaDeviceSynchronize();
  if (P->dmem) cudaFree(P->dmem);
  if (P->scratch) cudaFree(P->scratch);
  if (P->tc.trace) cudaFree(P->tc.trace);
  if (P->scratch_ev) cudaEventDestroy(P->scratch_ev);
  if (P->stage) cudaFree(P->stage);
  for (auto& s : P->hs)
    if (s) cudaStreamDestroy(s);
  if (P->hev) cudaEventDestroy(P->hev);
  cudaSetDevice(prev);
  delete P;
  return ITLUMM_OK;
}

extern "C" itlumm_status itlumm_plan_set_algo(itlumm_plan P, itlumm_algo algo) {
  g_err.clear();
  if (!P) return fail(ITLUMM_EINVAL, "plan is NULL");
  if (algo != ITLUMM_ALGO_AUTO && algo != ITLUMM_ALGO_SIMT && algo != ITLUMM_ALGO_TC && algo != ITLUMM_ALGO_TC_PIPE)
    return fail(ITLUMM_EINVAL, "bad algo %d", (int)algo);
  P->algo = algo;
  return ITLUMM_OK;
}

extern "C" itlumm_status itlumm_plan_set_summation(itlumm_plan P, itlumm_summation s) {
  g_err.clear();
  if (!P) return fail(ITLUMM_EINVAL, "plan is NULL");
  if (s != ITLUMM_SUM_EXACT && s != ITLUMM_SUM_AVG16) return fail(ITLUMM_EINVAL, "bad summation %d", (int)s);
  if (s == ITLUMM_SUM_AVG16 && P->C % 16 != 0)
    return fail(ITLUMM_EINVAL, "avg16 summation needs C %% 16 == 0 (C = %d)", P->C);
  P->summation = s;
  return ITLUMM_OK;
}

extern "C" itlumm_status itlumm_plan_set_onehot(itlumm_plan P, itlumm_onehot o) {
  g_err.clear();
  if (!P) return fail(ITLUMM_EINVAL, "plan is NULL");
  if (o != ITLUMM_ONEHOT_AUTO && o != ITLUMM_ONEHOT_DENSE && o != ITLUMM_ONEHOT_SPARSE24)
    return fail(ITLUMM_EINVAL, "bad onehot %d", (int)o);
  if (o == ITLUMM_ONEHOT_SPARSE24 && !P->tcs.ok)
    return fail(ITLUMM_EUNSUPPORTED, "2:4-sparse one-hot tiling unsupported for this plan: %s", P->tcs.why);
  P->onehot = o;
  return ITLUMM_OK;
}

extern "C" itlumm_status itlumm_plan_info(itlumm_plan P, int32_t* D, int32_t* C, int32_t* M, int64_t* lut_bytes) {
  g_err.clear();
  if (!P) return fail(ITLUMM_EINVAL, "plan is NULL");
  if (D) *D = P->D;
  if (C) *C = P->C;
  if (M) *M = P->M;
  if (lut_bytes) *lut_bytes = (int64_t)16 * P->C * P->M;
  return ITLUMM_OK;
}

// ------------------------------------------------------------------------------ launches
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev); else prev = -1;
  }
  ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

static itlumm_status check_A(itlumm_plan P, const void* A, itlumm_dtype dtype, int64_t lda, int64_t N) {
  if (!P) return fail(ITLUMM_EINVAL, "plan is NULL");
  if (N < 0) return fail(ITLUMM_EINVAL, "N < 0");
  if (dtype != ITLUMM_F32 && dtype != ITLUMM_BF16) return fail(ITLUMM_EINVAL, "bad dtype %d", (int)dtype);
  if (N > 0 && !A) return fail(ITLUMM_EINVAL, "A is NULL");
  if (lda < P->D) return fail(ITLUMM_ESHAPE, "lda (%lld) < D (%d)", (long long)lda, P->D);
  return ITLUMM_OK;
}

// A device pointer the caller passes must be device (or managed) memory of the plan's device.
static itlumm_status check_dev(itlumm_plan P, const void* ptr, const char* what) {
  cudaPointerAttributes at{};
  cudaError_t e = cudaPointerGetAttributes(&at, ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(ITLUMM_EINVAL, "%s: not a CUDA-visible pointer (%s)", what, cudaGetErrorString(e));
  }
  if (at.type == cudaMemoryTypeManaged || (at.type == cudaMemoryTypeDevice && at.device == P->device)) return ITLUMM_OK;
  return fail(ITLUMM_EINVAL, "%s is not device memory of the plan's device %d (memory type %d, device %d)", what,
              P->device, (int)at.type, at.device);
}

// Rows per stage R and ring depth S of the streaming encoder for rows of rb bytes, or false if
// the rows cannot be bulk-copied.
static bool enc_tiling(itlumm_plan P, int64_t rb, int consumer_warps, int* Rout, int* Sout,
                       int inflight_override_kb = 0, int max_stages = 8, int64_t N = 0) {
  // ~24 KB stages and ~100 KB in flight per SM: the measured optimum of a cfg2 sweep (more
  // bytes in flight lowered DRAM efficiency: 6.1 TB/s at 4 x 25 KB vs 5.5 TB/s at 6 x 31 KB,
  // profiles/r01/encode_stage_sweep.txt).  Developer overrides (not ABI):
  // ITLUMM_ENC_STAGE_KB, ITLUMM_ENC_INFLIGHT_KB.
  // 48 KB stages where the consumers are compute-heavy (C >= 128: the per-tile handshake is amortised
  // over twice the rows; D=592 C=256 encode 294 -> 263 us) and, with 16 consumer warps, wherever the
  // call has a full wave of 48 KB tiles (cfg2 packed encode 12.3 -> 9.9 us, row-major 32.1 -> 30.8 us,
  // cfg3 C=128 packed 34.7 -> 24.9 us, measured with 16 warps; tools/gpu_encwarps.sh)
  static const int stage_kb_env = getenv("ITLUMM_ENC_STAGE_KB") ? atoi(getenv("ITLUMM_ENC_STAGE_KB")) : 0;
  const bool big = P->C >= 128 || N * rb >= (int64_t)P->num_sms * 48 * 1024;
  const int stage_kb = stage_kb_env > 0 ? stage_kb_env : (big ? 48 : 24);
  static const int inflight_kb = getenv("ITLUMM_ENC_INFLIGHT_KB") ? atoi(getenv("ITLUMM_ENC_INFLIGHT_KB")) : 100;
  if (rb > 64 * 1024) return false;
  const int ngrp = (P->C + 31) / 32;
  const int want = std::min(8, (consumer_warps + ngrp - 1) / ngrp);
  int R = (int)std::max<int64_t>(want, ((int64_t)stage_kb * 1024) / rb);
  if ((int64_t)((R + want - 1) / want * want) * rb <= 64 * 1024) R = (R + want - 1) / want * want;
  if ((int64_t)R * rb > 64 * 1024) R = (int)std::max<int64_t>(1, (64 * 1024) / rb);
  const int64_t infl = inflight_override_kb > 0 ? inflight_override_kb : inflight_kb;
  int S = (int)std::max<int64_t>(2, std::min<int64_t>(max_stages, (infl * 1024 + R * rb / 2) / (R * rb)));
  while (S >= 2 && enc_smem_bytes(P->C, R, S, (int)rb) > 200 * 1024) --S;
  if (S < 2) return false;
  *Rout = R;
  *Sout = S;
  return true;
}

// Streaming encode (k_encode_rows) when the rows can be bulk-copied (16-byte aligned rows whose
// byte length is a multiple of 16) and a 2-stage ring fits in shared memory; otherwise the
// per-thread gather kernel k_encode.
static itlumm_status launch_encode(itlumm_plan P, const void* A, itlumm_dtype dtype, int64_t lda,
                                   int64_t N, uint8_t* codes, int64_t ldc, cudaStream_t s, bool pdl = false,
                                   bool pdl_dep = false) {
  const int es = dtype == ITLUMM_BF16 ? 2 : 4;
  const int64_t rb = (int64_t)P->D * es;
  const bool aligned = ((uintptr_t)A % 16 == 0) && ((lda * es) % 16 == 0) && (rb % 16 == 0);
  // Stream whole rows when the split columns touch most of a row's DRAM lines (cfg2: 98%); gather
  // the columns per thread when they touch few of them (cfg4 C=16 layer 1: 64 of 3072 columns).
  const bool sparse_cols = P->seg_frac[dtype == ITLUMM_BF16 ? 1 : 0] < 0.6;
  int R = 0, S = 0;
  // 16 consumer warps: with 8 the encoder was latency-bound (ncu: 14% warps active, 32% issue) on
  // split-packed rows, whose tree walks per byte are 6x those of row-major cfg2 rows.  Developer
  // override: ITLUMM_ENC_WARPS.
  static const int enc_warps_env = getenv("ITLUMM_ENC_WARPS") ? atoi(getenv("ITLUMM_ENC_WARPS")) : 0;
  const int enc_warps = enc_warps_env > 0 ? std::min(enc_warps_env, kEncMaxConsumerWarps) : kEncConsumerWarps;
  if (aligned && !sparse_cols && enc_tiling(P, rb, enc_warps, &R, &S, 0, 8, N)) {
    {
      EncArgs g{};
      g.A = A; g.lda = lda; g.N = N; g.codes = codes; g.ldc = ldc;
      g.R = R; g.S = S; g.row_bytes = (int)rb; g.contiguous = lda == P->D; g.pdl = pdl ? 1 : 0;
      g.packed = P->packed ? 1 : 0;
      // register-threshold consumer: split-packed rows (cfg2 packed encode 19.7 -> 11.6 us) and
      // C > 32 (cfg4 C=256 MLP 12.8 -> 10.7 ms); row-major C = 32 keeps the shared-memory walk
      // (31.8 vs 32.5 us).  Developer override: ITLUMM_ENC_FIXED (0 never, 1 auto, 2 always).
      static const int fixed_env = getenv("ITLUMM_ENC_FIXED") ? atoi(getenv("ITLUMM_ENC_FIXED")) : 1;
      g.fixed_ok = fixed_env == 2 || (fixed_env == 1 && (P->packed || P->C > 32));
      // Row reads are marked L2 evict_first: streamed once, they should not displace what the step
      // reuses (cfg2 step 62.9 -> 58.9 us, cfg3 C=64 168.8 -> 158.4 us; profiles/r01/l2_hint_sweep.jsonl).
      // Developer override: ITLUMM_A_HINT (0 none, 1 evict_first, 2 evict_last, 3/4 evict_first on 1/2 or 1/4).
      static const int a_hint = getenv("ITLUMM_A_HINT") ? atoi(getenv("ITLUMM_A_HINT")) : 1;
      g.a_hint = a_hint;
      g.span = P->tc.trace ? P->tc.trace + (size_t)16 * 4 * kTraceEv : nullptr;
      const int64_t ntiles = (N + R - 1) / R;
      const unsigned grid = (unsigned)std::min<int64_t>(ntiles, P->num_sms);
      const size_t smem = enc_smem_bytes(P->C, R, S, (int)rb);
      // pdl_dep: a programmatic dependent of the previous kernel on the stream (the prologue
      // overlaps its tail; griddepcontrol.wait before any read of A).  Only for single-wave
      // encodes, which are launch-latency bound (cfg1: 7.67 -> 6.35 us per call); multi-wave ones
      // got slower (cfg2 58.8 -> 63.6 us; profiles/r01/encoder_pdl.jsonl).  Developer override:
      // ITLUMM_ENC_PDL (0 never, 1 single-wave, 2 always).
      static const int dep_env = getenv("ITLUMM_ENC_PDL") ? atoi(getenv("ITLUMM_ENC_PDL")) : 1;
      g.pdl_wait = (pdl_dep && (dep_env == 2 || (dep_env == 1 && ntiles <= P->num_sms))) ? 1 : 0;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(32 * (1 + enc_warps));
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = g.pdl_wait ? 1 : 0;
      const bool wide = P->C >= 32;
      if (dtype == ITLUMM_F32)
        CUDA_TRY(cudaLaunchKernelEx(&cfg, wide ? k_encode_rows<float, true> : k_encode_rows<float, false>, P->dp, g));
      else
        CUDA_TRY(cudaLaunchKernelEx(&cfg, wide ? k_encode_rows<uint16_t, true> : k_encode_rows<uint16_t, false>, P->dp, g));
      CUDA_TRY(cudaGetLastError());
      g_launches = 1;
      return ITLUMM_OK;
    }
  }
  const int64_t nb = (P->C + 1) / 2;
  const int64_t total = N * nb;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)P->num_sms * 32);
  if (dtype == ITLUMM_F32)
    k_encode<float><<<(unsigned)blocks, 256, 0, s>>>(P->dp, (const float*)A, lda, N, codes, ldc);
  else
    k_encode<uint16_t><<<(unsigned)blocks, 256, 0, s>>>(P->dp, (const uint16_t*)A, lda, N, codes, ldc);
  CUDA_TRY(cudaGetLastError());
  g_launches = 1;
  return ITLUMM_OK;
}

extern "C" itlumm_status itlumm_encode(itlumm_plan P, const void* A, itlumm_dtype dtype, int64_t lda,
                                       int64_t N, uint8_t* codes, int64_t ldc, void* stream) {
  g_err.clear();
  g_launches = 0;
  itlumm_status st = check_A(P, A, dtype, lda, N);
  if (st != ITLUMM_OK) return st;
  if (ldc < (P->C + 1) / 2) return fail(ITLUMM_ESHAPE, "ldc (%lld) < ceil(C/2) (%d)", (long long)ldc, (P->C + 1) / 2);
  if (N == 0) return ITLUMM_OK;
  if (!codes) return fail(ITLUMM_EINVAL, "codes is NULL");
  if ((st = check_dev(P, A, "A")) != ITLUMM_OK || (st = check_dev(P, codes, "codes")) != ITLUMM_OK) return st;
  DeviceGuard dg(P->device);
  return launch_encode(P, A, dtype, lda, N, codes, ldc, (cudaStream_t)stream);
}

// The 1-CTA tensor-core tiling in use: dense (AUTO, DENSE) or 2:4-sparse one-hot (SPARSE24).
static const TcPlan& tcp(itlumm_plan P) { return P->onehot == ITLUMM_ONEHOT_SPARSE24 ? P->tcs : P->tc; }

// Tensor-core accumulate of codes (a3' + a4): a streamed LUT runs the CTA-pair kernel k_tcp (dense
// or 2:4-sparse one-hot), a resident LUT the 1-CTA k_tc.  Developer knob (not ABI): ITLUMM_PAIR=0
// keeps streamed LUTs on k_tc.
static itlumm_status launch_tc_acc(itlumm_plan P, const TcArgs& a, cudaStream_t s, bool pdl) {
  static const bool pair_on = !(getenv("ITLUMM_PAIR") && atoi(getenv("ITLUMM_PAIR")) == 0);
  const TcPlan& t = tcp(P);
  if (pair_on && t.ok && t.stream_b) {
    const TcpPlan& pp = P->onehot == ITLUMM_ONEHOT_SPARSE24 ? P->pair_sp : P->pair_dn;
    if (pp.ok) {
      const itlumm_status st = tcp_launch(pp, P->dp, a, s, pdl);
      if (st != ITLUMM_EUNSUPPORTED) return st;
    }
  }
  return tc_launch(t, P->dp, false, false, a, s, pdl);
}

static bool use_tc(itlumm_plan P) {
  if (P->algo == ITLUMM_ALGO_SIMT || P->summation != ITLUMM_SUM_EXACT) return false;
  if (P->algo == ITLUMM_ALGO_TC || P->algo == ITLUMM_ALGO_TC_PIPE) return true;
  return tc_preferred(tcp(P), P->simt.MS != 0);
}

// The fused call runs as encode -> TC accumulate when asked to (TC_PIPE), or under AUTO when
// the tensor-core tiling splits M over several CTAs (a fused kernel would repeat the gather
// and the tree walks once per M slice).
static bool use_pipe(itlumm_plan P) {
  if (!tcp(P).ok || P->summation != ITLUMM_SUM_EXACT) return false;
  if (P->algo == ITLUMM_ALGO_TC_PIPE) return true;
  // AUTO pipes every tensor-core shape through the streaming encoder: a streamed LUT has no fused
  // TC kernel, with several slices a fused kernel would repeat the gather per slice, and even with
  // one slice the fused kernel's per-thread gather is latency-bound (cfg1: 10.0 us fused vs 6.6 us
  // encode + accumulate)
  return P->algo == ITLUMM_ALGO_AUTO;
}

static itlumm_status launch_lut(itlumm_plan P, bool fused, const void* A, itlumm_dtype dtype, int64_t lda,
                                const uint8_t* codes, int64_t ldc, int64_t N, int32_t* acc, int64_t ldacc,
                                float* out, int64_t ldo, itlumm_epilogue epi, cudaStream_t s) {
  if (use_tc(P)) {
    const TcPlan& t = tcp(P);
    if (!t.ok) return fail(ITLUMM_EUNSUPPORTED, "tensor-core path unsupported for this plan: %s", t.why);
    TcArgs a{};
    a.A = A; a.lda = lda; a.codes = codes; a.ldc = ldc; a.N = N; a.acc = acc; a.ldacc = ldacc;
    a.out = out; a.ldo = ldo; a.relu = epi == ITLUMM_EPI_RELU;
    a.packed = P->packed ? 1 : 0;
    itlumm_status st = fused ? tc_launch(t, P->dp, true, dtype == ITLUMM_BF16, a, s) : launch_tc_acc(P, a, s, false);
    if (st == ITLUMM_OK) {
      g_launches = 1;
      return ITLUMM_OK;
    }
    // AUTO never fails on a shape the CUDA-core kernels take (e.g. a streamed LUT with codes rows
    // that are not 16-byte multiples): fall through to SIMT; an explicit TC request reports the error
    if (!(st == ITLUMM_EUNSUPPORTED && P->algo == ITLUMM_ALGO_AUTO && P->simt.MS != 0))
      return fail(st, "%s", tc_last_msg());
  }
  const SimtCfg& c = P->simt;
  if (c.MS == 0) return fail(ITLUMM_EUNSUPPORTED, "SIMT LUT kernel: C = %d too large for a resident LUT slice", P->C);
  LutArgs g{};
  g.A = A; g.lda = lda; g.codes = codes; g.ldc = ldc; g.N = N;
  g.acc = acc; g.ldacc = ldacc; g.out = out; g.ldo = ldo;
  g.relu = epi == ITLUMM_EPI_RELU;
  const bool out_al = !out || (((uintptr_t)out % 16) == 0 && ldo % 4 == 0);
  const bool acc_al = !acc || (((uintptr_t)acc % 16) == 0 && ldacc % 4 == 0);
  g.vec_out = out_al && acc_al;
  g.R = c.R; g.RPT = c.RPT; g.S = c.S; g.G = c.G; g.one = 1u;
  const int64_t ntiles = (N + c.R - 1) / c.R;
  int grid = fused ? c.grid_fused : c.grid_codes;
  const int64_t maxgrid = (int64_t)c.G * ntiles;
  if (grid > maxgrid) grid = (int)maxgrid;
  lut_kernel_t k;
  if (P->summation == ITLUMM_SUM_AVG16)
    k = fused ? (dtype == ITLUMM_BF16 ? pick_lut_kernel<true, uint16_t, true>(c.MS)
                                     : pick_lut_kernel<true, float, true>(c.MS))
              : pick_lut_kernel<false, float, true>(c.MS);
  else
    k = fused ? (dtype == ITLUMM_BF16 ? pick_lut_kernel<true, uint16_t>(c.MS)
                                      : pick_lut_kernel<true, float>(c.MS))
              : pick_lut_kernel<false, float>(c.MS);
  k<<<grid, kLutThreads, fused ? c.smem_fused : c.smem_codes, s>>>(P->dp, g);
  CUDA_TRY(cudaGetLastError());
  g_launches = 1;
  return ITLUMM_OK;
}

// encode -> codes scratch (L2-resident) -> TC accumulate, chunked by the scratch height.
static itlumm_status launch_pipe(itlumm_plan P, const void* A, itlumm_dtype dtype, int64_t lda, int64_t N,
                                 float* out, int64_t ldo, itlumm_epilogue epi, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(P->scratch_mu);
  // Calls on different streams share the plan's code scratch: order them through an event.  A
  // stream being captured into a CUDA graph is ordered by the graph itself (an event recorded
  // outside the capture cannot be waited on inside it).
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CUDA_TRY(cudaStreamIsCapturing(s, &cap));
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  if (P->scratch_used && !capturing) CUDA_TRY(cudaStreamWaitEvent(s, P->scratch_ev, 0));
  const size_t es = dtype == ITLUMM_BF16 ? 2 : 4;
  int32_t launches = 0;
  for (int64_t r0 = 0; r0 < N; r0 += P->scratch_rows) {
    const int64_t rows = std::min<int64_t>(P->scratch_rows, N - r0);
    const void* Ar = (const uint8_t*)A + (size_t)r0 * lda * es;
    itlumm_status st = launch_encode(P, Ar, dtype, lda, rows, P->scratch, P->scratch_ldc, s, true, true);
    if (st != ITLUMM_OK) return st;
    TcArgs a{};
    a.codes = P->scratch; a.ldc = P->scratch_ldc; a.N = rows;
    a.out = out + (size_t)r0 * ldo; a.ldo = ldo; a.relu = epi == ITLUMM_EPI_RELU;
    st = launch_tc_acc(P, a, s, true);
    if (st != ITLUMM_OK) return fail(st, "%s", tc_last_msg());
    launches += 2;
  }
  if (!capturing) {
    CUDA_TRY(cudaEventRecord(P->scratch_ev, s));
    P->scratch_used = true;
  }
  g_launches = launches;
  return ITLUMM_OK;
}

extern "C" itlumm_status itlumm_lut_accumulate(itlumm_plan P, const uint8_t* codes, int64_t ldc, int64_t N,
                                               int32_t* acc, int64_t ldacc, float* out, int64_t ldo,
                                               itlumm_epilogue epi, void* stream) {
  g_err.clear();
  g_launches = 0;
  if (!P) return fail(ITLUMM_EINVAL, "plan is NULL");
  if (N < 0) return fail(ITLUMM_EINVAL, "N < 0");
  if (epi != ITLUMM_EPI_NONE && epi != ITLUMM_EPI_RELU) return fail(ITLUMM_EINVAL, "bad epilogue");
  if (ldc < (P->C + 1) / 2) return fail(ITLUMM_ESHAPE, "ldc (%lld) < ceil(C/2)", (long long)ldc);
  if (acc && ldacc < P->M) return fail(ITLUMM_ESHAPE, "ldacc < M");
  if (out && ldo < P->M) return fail(ITLUMM_ESHAPE, "ldo < M");
  if (N == 0) return ITLUMM_OK;
  if (!codes) return fail(ITLUMM_EINVAL, "codes is NULL");
  if (!acc && !out) return fail(ITLUMM_EINVAL, "acc and out are both NULL");
  itlumm_status st;
  if ((st = check_dev(P, codes, "codes")) != ITLUMM_OK) return st;
  if (acc && (st = check_dev(P, acc, "acc")) != ITLUMM_OK) return st;
  if (out && (st = check_dev(P, out, "out")) != ITLUMM_OK) return st;
  DeviceGuard dg(P->device);
  return launch_lut(P, false, nullptr, ITLUMM_F32, 0, codes, ldc, N, acc, ldacc, out, ldo, epi, (cudaStream_t)stream);
}

extern "C" itlumm_status itlumm_amm(itlumm_plan P, const void* A, itlumm_dtype dtype, int64_t lda, int64_t N,
                                    float* out, int64_t ldo, itlumm_epilogue epi, void* stream) {
  g_err.clear();
  g_launches = 0;
  itlumm_status st = check_A(P, A, dtype, lda, N);
  if (st != ITLUMM_OK) return st;
  if (epi != ITLUMM_EPI_NONE && epi != ITLUMM_EPI_RELU) return fail(ITLUMM_EINVAL, "bad epilogue");
  if (ldo < P->M) return fail(ITLUMM_ESHAPE, "ldo (%lld) < M (%d)", (long long)ldo, P->M);
  if (N == 0) return ITLUMM_OK;
  if (!out) return fail(ITLUMM_EINVAL, "out is NULL");
  if ((st = check_dev(P, A, "A")) != ITLUMM_OK || (st = check_dev(P, out, "out")) != ITLUMM_OK) return st;
  DeviceGuard dg(P->device);
  if (use_pipe(P)) return launch_pipe(P, A, dtype, lda, N, out, ldo, epi, (cudaStream_t)stream);
  return launch_lut(P, true, A, dtype, lda, nullptr, 0, N, nullptr, 0, out, ldo, epi, (cudaStream_t)stream);
}

extern "C" itlumm_status itlumm_amm_host(itlumm_plan P, const void* A_host, itlumm_dtype dtype, int64_t lda,
                                         int64_t N, float* out_host, int64_t ldo, itlumm_epilogue epi,
                                         void* stream) {
  g_err.clear();
  g_launches = 0;
  itlumm_status st = check_A(P, A_host, dtype, lda, N);
  if (st != ITLUMM_OK) return st;
  if (epi != ITLUMM_EPI_NONE && epi != ITLUMM_EPI_RELU) return fail(ITLUMM_EINVAL, "bad epilogue");
  if (ldo < P->M) return fail(ITLUMM_ESHAPE, "ldo (%lld) < M (%d)", (long long)ldo, P->M);
  if (N == 0) return ITLUMM_OK;
  if (!out_host) return fail(ITLUMM_EINVAL, "out_host is NULL");
  std::lock_guard<std::mutex> lk(P->host_mu);
  DeviceGuard dg(P->device);
  const size_t es = dtype == ITLUMM_BF16 ? 2 : 4;
  const size_t row_in = (size_t)P->D * es, row_out = (size_t)P->M * 4;
  // chunk of rows per pipeline stage: ~16 MB of input, at least 1024 rows; 3 stages in a ring so
  // that the H2D of chunk i+1, the kernels of chunk i and the D2H of chunk i-1 overlap
  constexpr int kStages = 3;
  int64_t chunk = std::max<int64_t>(1024, (int64_t)((16u << 20) / row_in));
  chunk = std::min<int64_t>(chunk, N);
  const size_t in_b = ((size_t)chunk * row_in + 255) & ~(size_t)255, out_b = ((size_t)chunk * row_out + 255) & ~(size_t)255;
  const size_t need = kStages * (in_b + out_b);
  if (P->stage_bytes < need) {
    if (P->stage) { cudaDeviceSynchronize(); cudaFree(P->stage); P->stage = nullptr; P->stage_bytes = 0; }
    if (cudaMalloc(&P->stage, need) != cudaSuccess) return fail(ITLUMM_ENOMEM, "staging cudaMalloc(%zu)", need);
    P->stage_bytes = need;
  }
  for (auto& s : P->hs)
    if (!s) CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  if (!P->hev) CUDA_TRY(cudaEventCreateWithFlags(&P->hev, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(P->hev, (cudaStream_t)stream));
  for (auto& s : P->hs) CUDA_TRY(cudaStreamWaitEvent(s, P->hev, 0));
  int32_t launches = 0;
  for (int64_t r0 = 0, i = 0; r0 < N; r0 += chunk, ++i) {
    const int64_t rows = std::min<int64_t>(chunk, N - r0);
    cudaStream_t s = P->hs[i % kStages];
    uint8_t* dA = (uint8_t*)P->stage + (i % kStages) * (in_b + out_b);
    float* dO = (float*)(dA + in_b);
    const uint8_t* hA = (const uint8_t*)A_host + (size_t)r0 * lda * es;
    if ((size_t)lda * es == row_in)
      CUDA_TRY(cudaMemcpyAsync(dA, hA, (size_t)rows * row_in, cudaMemcpyHostToDevice, s));
    else
      CUDA_TRY(cudaMemcpy2DAsync(dA, row_in, hA, (size_t)lda * es, row_in, rows, cudaMemcpyHostToDevice, s));
    if (use_pipe(P)) {
      st = launch_pipe(P, dA, dtype, P->D, rows, dO, P->M, epi, s);
    } else {
      st = launch_lut(P, true, dA, dtype, P->D, nullptr, 0, rows, nullptr, 0, dO, P->M, epi, s);
    }
    if (st != ITLUMM_OK) return st;
    launches += g_launches;
    if (ldo == P->M)
      CUDA_TRY(cudaMemcpyAsync(out_host + (size_t)r0 * ldo, dO, (size_t)rows * row_out, cudaMemcpyDeviceToHost, s));
    else
      CUDA_TRY(cudaMemcpy2DAsync(out_host + (size_t)r0 * ldo, (size_t)ldo * 4, dO, row_out, row_out, rows,
                                 cudaMemcpyDeviceToHost, s));
  }
  for (auto& s : P->hs) CUDA_TRY(cudaStreamSynchronize(s));
  g_launches = launches;
  return ITLUMM_OK;
}

// ------------------------------------------------------------------------------ MLP chaining
struct itlumm_mlp_s {
  int device = 0;
  std::vector<itlumm_plan> plans;
  std::vector<itlumm_epilogue> epis;
  std::vector<int> width;     // output columns computed by layer l
  std::vector<int> ld;        // row stride of layer l's intermediate buffer (width rounded up to 4)
  std::vector<float*> buf;    // intermediate buffers, chunk rows each (all but the last layer)
  int64_t chunk = 262144, buf_rows = 0;
  // host API staging (itlumm_mlp_forward_host): 2 input + 2 output slots, copy streams, events
  std::mutex host_mu;
  void* stage = nullptr;
  size_t stage_bytes = 0;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev[8] = {};
};

extern "C" itlumm_status itlumm_mlp_destroy(itlumm_mlp m) {
  g_err.clear();
  if (!m) return ITLUMM_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(m->device);
  cudaDeviceSynchronize();
  for (auto* b : m->buf) if (b) cudaFree(b);
  if (m->stage) cudaFree(m->stage);
  if (m->h2d) cudaStreamDestroy(m->h2d);
  if (m->d2h) cudaStreamDestroy(m->d2h);
  for (auto& e : m->ev) if (e) cudaEventDestroy(e);
  for (auto p : m->plans) if (p) itlumm_plan_destroy(p);
  cudaSetDevice(prev);
  delete m;
  return ITLUMM_OK;
}

extern "C" itlumm_status itlumm_mlp_create(const itlumm_params* layers, const itlumm_epilogue* epis,
                                           int32_t n_layers, int cuda_device, itlumm_mlp* out) {
  g_err.clear();
  if (!out) return fail(ITLUMM_EINVAL, "out is NULL");
  *out = nullptr;
  if (!layers || !epis || n_layers < 1) return fail(ITLUMM_EINVAL, "layers/epis NULL or n_layers < 1");
  for (int l = 0; l + 1 < n_layers; ++l)
    if (layers[l + 1].D != layers[l].M)
      return fail(ITLUMM_ESHAPE, "layer %d has D = %d but layer %d has M = %d", l + 1, layers[l + 1].D, l, layers[l].M);
  for (int l = 0; l < n_layers; ++l)
    if (epis[l] != ITLUMM_EPI_NONE && epis[l] != ITLUMM_EPI_RELU) return fail(ITLUMM_EINVAL, "bad epilogue of layer %d", l);
  // columns of layer l's output that layer l+1 splits on (sorted, distinct)
  std::vector<std::vector<int32_t>> need(n_layers);
  for (int l = 0; l + 1 < n_layers; ++l) {
    const itlumm_params& q = layers[l + 1];
    if (!q.split_dim || q.C < 1 || q.C > q.D) return fail(ITLUMM_EINVAL, "layer %d: bad split_dim/C", l + 1);
    std::vector<int32_t> bnd(q.C + 1);
    if (q.boundaries) {
      for (int c = 0; c <= q.C; ++c) bnd[c] = q.boundaries[c];
    } else {
      const int qq = q.D / q.C, r = q.D % q.C;
      bnd[0] = 0;
      for (int c = 0; c < q.C; ++c) bnd[c + 1] = bnd[c] + qq + (c < r ? 1 : 0);
    }
    std::vector<char> used(q.D, 0);
    for (int c = 0; c < q.C; ++c)
      for (int t = 0; t < kLevels; ++t) {
        const int sd = q.split_dim[c * 4 + t];
        const int i = bnd[c] + sd;
        if (sd < 0 || i < bnd[c] || i >= bnd[c + 1] || i >= q.D) return fail(ITLUMM_EINVAL, "layer %d: split_dim out of range", l + 1);
        const int col = q.perm ? q.perm[i] : i;
        if (col < 0 || col >= q.D) return fail(ITLUMM_EINVAL, "layer %d: bad perm", l + 1);
        used[col] = 1;
      }
    for (int i = 0; i < q.D; ++i) if (used[i]) need[l].push_back(i);
  }
  itlumm_mlp_s* m = new (std::nothrow) itlumm_mlp_s();
  if (!m) return fail(ITLUMM_ENOMEM, "host allocation failed");
  m->device = cuda_device;
  m->plans.assign(n_layers, nullptr);
  m->epis.assign(epis, epis + n_layers);
  m->width.assign(n_layers, 0);
  m->ld.assign(n_layers, 0);
  for (int l = 0; l < n_layers; ++l) {
    PlanView v;
    const bool last = l + 1 == n_layers;
    if (!last) { v.out_cols = need[l].data(); v.n_out = (int)need[l].size(); }
    std::vector<int32_t> in_map;
    if (l > 0) {
      in_map.assign(layers[l].D, -1);
      for (size_t j = 0; j < need[l - 1].size(); ++j) in_map[need[l - 1][j]] = (int32_t)j;
      v.in_map = in_map.data();
      v.D_in = m->ld[l - 1];
    }
    itlumm_status st = plan_create_impl(&layers[l], cuda_device, v, &m->plans[l]);
    if (st != ITLUMM_OK) {
      std::string msg = "layer " + std::to_string(l) + ": " + g_err;
      itlumm_mlp_destroy(m);
      return fail(st, "%s", msg.c_str());
    }
    m->width[l] = last ? layers[l].M : (int)need[l].size();
    m->ld[l] = (m->width[l] + 3) & ~3;        // 16-byte rows: bulk-copyable, TMA-storable
  }
  *out = m;
  return ITLUMM_OK;
}

extern "C" itlumm_status itlumm_mlp_info(itlumm_mlp m, int32_t* n_layers, int32_t* widths) {
  g_err.clear();
  if (!m) return fail(ITLUMM_EINVAL, "mlp is NULL");
  if (n_layers) *n_layers = (int32_t)m->plans.size();
  if (widths) for (size_t l = 0; l < m->plans.size(); ++l) widths[l] = m->width[l];
  return ITLUMM_OK;
}

extern "C" itlumm_status itlumm_mlp_forward(itlumm_mlp m, const void* A, itlumm_dtype dtype, int64_t lda,
                                            int64_t N, float* out, int64_t ldo, void* stream) {
  g_err.clear();
  g_launches = 0;
  if (!m) return fail(ITLUMM_EINVAL, "mlp is NULL");
  const int L = (int)m->plans.size();
  itlumm_status st = check_A(m->plans[0], A, dtype, lda, N);
  if (st != ITLUMM_OK) return st;
  if (ldo < m->width[L - 1]) return fail(ITLUMM_ESHAPE, "ldo (%lld) < M (%d)", (long long)ldo, m->width[L - 1]);
  if (N == 0) return ITLUMM_OK;
  if (!out) return fail(ITLUMM_EINVAL, "out is NULL");
  if ((st = check_dev(m->plans[0], A, "A")) != ITLUMM_OK || (st = check_dev(m->plans[0], out, "out")) != ITLUMM_OK) return st;
  DeviceGuard dg(m->device);
  const int64_t rows_max = std::min<int64_t>(m->chunk, N);
  if (m->buf_rows < rows_max) {
    if (m->buf_rows) cudaDeviceSynchronize();
    for (auto*& b : m->buf) { if (b) cudaFree(b); b = nullptr; }
    m->buf.assign(L > 1 ? L - 1 : 0, nullptr);
    for (int l = 0; l + 1 < L; ++l)
      if (cudaMalloc(&m->buf[l], (size_t)rows_max * m->ld[l] * 4) != cudaSuccess) {
        for (auto*& b : m->buf) { if (b) cudaFree(b); b = nullptr; }
        m->buf_rows = 0;
        return fail(ITLUMM_ENOMEM, "intermediate buffers (%lld rows)", (long long)rows_max);
      }
    m->buf_rows = rows_max;
  }
  const size_t es = dtype == ITLUMM_BF16 ? 2 : 4;
  int32_t launches = 0;
  for (int64_t r0 = 0; r0 < N; r0 += m->chunk) {
    const int64_t rows = std::min<int64_t>(m->chunk, N - r0);
    const void* in = (const uint8_t*)A + (size_t)r0 * lda * es;
    itlumm_dtype dt = dtype;
    int64_t ld_in = lda;
    for (int l = 0; l < L; ++l) {
      const bool last = l + 1 == L;
      float* o = last ? out + (size_t)r0 * ldo : m->buf[l];
      const int64_t ld_o = last ? ldo : m->ld[l];
      st = itlumm_amm(m->plans[l], in, dt, ld_in, rows, o, ld_o, m->epis[l], stream);
      if (st != ITLUMM_OK) {
        std::string msg = "layer " + std::to_string(l) + ": " + g_err;
        return fail(st, "%s", msg.c_str());
      }
      launches += g_launches;
      in = o; dt = ITLUMM_F32; ld_in = ld_o;
    }
  }
  g_launches = launches;
  return ITLUMM_OK;
}

extern "C" itlumm_status itlumm_mlp_forward_host(itlumm_mlp m, const void* A_host, itlumm_dtype dtype, int64_t lda,
                                                 int64_t N, float* out_host, int64_t ldo, void* stream) {
  g_err.clear();
  g_launches = 0;
  if (!m) return fail(ITLUMM_EINVAL, "mlp is NULL");
  const int L = (int)m->plans.size();
  itlumm_status st = check_A(m->plans[0], A_host, dtype, lda, N);
  if (st != ITLUMM_OK) return st;
  const int Mo = m->width[L - 1];
  if (ldo < Mo) return fail(ITLUMM_ESHAPE, "ldo (%lld) < M (%d)", (long long)ldo, Mo);
  if (N == 0) return ITLUMM_OK;
  if (!out_host) return fail(ITLUMM_EINVAL, "out_host is NULL");
  std::lock_guard<std::mutex> lk(m->host_mu);
  DeviceGuard dg(m->device);
  const size_t es = dtype == ITLUMM_BF16 ? 2 : 4;
  const int D = m->plans[0]->D;
  const size_t row_in = (size_t)D * es, row_out = (size_t)Mo * 4;
  // chunks of ~64 MB of input (at least 1024 rows) through 2 input and 2 output slots: the H2D of
  // chunk i+1 and the D2H of chunk i-1 overlap the forward of chunk i (forwards run in order on
  // `stream`, they share the MLP's intermediate buffers)
  int64_t chunk = std::max<int64_t>(1024, (int64_t)((64u << 20) / row_in));
  chunk = std::min<int64_t>(chunk, N);
  const size_t in_b = ((size_t)chunk * row_in + 255) & ~(size_t)255, out_b = ((size_t)chunk * row_out + 255) & ~(size_t)255;
  const size_t need = 2 * (in_b + out_b);
  if (m->stage_bytes < need) {
    if (m->stage) { cudaDeviceSynchronize(); cudaFree(m->stage); m->stage = nullptr; m->stage_bytes = 0; }
    if (cudaMalloc(&m->stage, need) != cudaSuccess) return fail(ITLUMM_ENOMEM, "staging cudaMalloc(%zu)", need);
    m->stage_bytes = need;
  }
  if (!m->h2d) CUDA_TRY(cudaStreamCreateWithFlags(&m->h2d, cudaStreamNonBlocking));
  if (!m->d2h) CUDA_TRY(cudaStreamCreateWithFlags(&m->d2h, cudaStreamNonBlocking));
  for (auto& e : m->ev)
    if (!e) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // ev[0..1] input slot loaded, ev[2..3] forward done (input slot free, output ready), ev[4..5]
  // output slot drained, ev[6] start
  cudaStream_t sc = (cudaStream_t)stream;
  CUDA_TRY(cudaEventRecord(m->ev[6], sc));
  CUDA_TRY(cudaStreamWaitEvent(m->h2d, m->ev[6], 0));
  CUDA_TRY(cudaStreamWaitEvent(m->d2h, m->ev[6], 0));
  int32_t launches = 0;
  for (int64_t r0 = 0, i = 0; r0 < N; r0 += chunk, ++i) {
    const int64_t rows = std::min<int64_t>(chunk, N - r0);
    const int s = (int)(i & 1);
    uint8_t* dA = (uint8_t*)m->stage + s * (in_b + out_b);
    float* dO = (float*)(dA + in_b);
    const uint8_t* hA = (const uint8_t*)A_host + (size_t)r0 * lda * es;
    if (i >= 2) CUDA_TRY(cudaStreamWaitEvent(m->h2d, m->ev[2 + s], 0));    // forward of chunk i-2 read the slot
    if ((size_t)lda * es == row_in)
      CUDA_TRY(cudaMemcpyAsync(dA, hA, (size_t)rows * row_in, cudaMemcpyHostToDevice, m->h2d));
    else
      CUDA_TRY(cudaMemcpy2DAsync(dA, row_in, hA, (size_t)lda * es, row_in, rows, cudaMemcpyHostToDevice, m->h2d));
    CUDA_TRY(cudaEventRecord(m->ev[s], m->h2d));
    CUDA_TRY(cudaStreamWaitEvent(sc, m->ev[s], 0));
    if (i >= 2) CUDA_TRY(cudaStreamWaitEvent(sc, m->ev[4 + s], 0));        // D2H of chunk i-2 drained the slot
    st = itlumm_mlp_forward(m, dA, dtype, D, rows, dO, Mo, sc);
    if (st != ITLUMM_OK) return st;
    launches += g_launches;
    CUDA_TRY(cudaEventRecord(m->ev[2 + s], sc));
    CUDA_TRY(cudaStreamWaitEvent(m->d2h, m->ev[2 + s], 0));
    if (ldo == Mo)
      CUDA_TRY(cudaMemcpyAsync(out_host + (size_t)r0 * ldo, dO, (size_t)rows * row_out, cudaMemcpyDeviceToHost, m->d2h));
    else
      CUDA_TRY(cudaMemcpy2DAsync(out_host + (size_t)r0 * ldo, (size_t)ldo * 4, dO, row_out, row_out, rows,
                                 cudaMemcpyDeviceToHost, m->d2h));
    CUDA_TRY(cudaEventRecord(m->ev[4 + s], m->d2h));
  }
  CUDA_TRY(cudaStreamSynchronize(m->d2h));
  CUDA_TRY(cudaStreamSynchronize(sc));
  g_launches = launches;
  return ITLUMM_OK;
}

// Developer timeline (not in the ABI header): with ITLUMM_TC_TRACE=1 at plan creation every TC
// launch of the plan records globaltimer stamps of CTAs 0..7 (producer K-block arrives, MMA tile
// starts and K-block commits, epilogue warp-0 tile start/end, codes loads); copy them out here.
extern "C" int itlumm_dbg_trace_copy(itlumm_plan P, uint64_t* host, int64_t n) {
  if (!P || !P->tc.trace || !host) return 1;
  const int64_t total = (int64_t)16 * 4 * kTraceEv + 4 * 512;
  cudaDeviceSynchronize();
  return cudaMemcpy(host, P->tc.trace, (size_t)std::min(n, total) * 8, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 2;
}

extern "C" int32_t itlumm_last_launch_count(void) { return g_launches; }
extern "C" const char* itlumm_last_error(void) { return g_err.c_str(); }
extern "C" int32_t itlumm_abi_version(void) { return ITLUMM_ABI_VERSION; }
