/* ORACLE — plain, slow, obviously-correct CPU implementation of the ITLUMM inference path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
 * leg may load this library.  It shares no code, header or constant with the CUDA library
 * (paper_2207_05808_b200/csrc); neither includes the other.
 *
 * Per row a:
 *   (1) a'[i] = a[perm[i]]                         permutation, reading R11 (gather)
 *       chunk c = a'[b[c] .. b[c+1])                contiguous subspaces
 *   (2) node = 0; for t = 0..3:                     "exactly 4 comparisons"
 *         v = chunk_c[split_dim[c][t]]
 *         node = 2*node + (v > thr[c][2^t - 1 + node])     (reading R1)
 *       code_c = node in [0,16)
 *   (3) acc[m] = sum_c q[c][code_c][m]              exact integer sum (reading R7)
 *   (4) y[m] = fmaf(scale[m], (float)acc[m], offtot[m]),
 *       offtot[m] = (float)((double)C*(double)offset[m] + (double)bias[m])   (reading R8)
 *       ReLU: y > 0 ? y : +0                       (reading R9)
 * bf16 inputs are widened exactly to fp32 first (reading R13).
 *
 * summation = 1 ("avg16", reading R22 — MADDNESS's "fast rounded 8-bit summation
 * over subspaces"): codebooks are taken in groups of 16 in index order (C % 16 == 0); per
 * output m a 4-level tree of rounding averages avg(a, b) = (a + b + 1) >> 1 over the group's 16
 * uint8 entries, pairs (0,1),(2,3),... at every level, gives a_g; acc[m] = sum_g a_g exactly.  The
 * tree over-estimates the group mean by +1 in expectation, so
 *   y[m] = fmaf(16*scale[m], (float)acc[m], offavg[m]),
 *   offavg[m] = (float)((double)C*offset[m] + bias[m] - 16*(C/16)*(double)scale[m]).
 * Compiled with -O2 -ffp-contract=off; fmaf is the only fused operation.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t r0, r1;
  int D, C, M, dtype, relu;
  const void* A;
  int64_t lda;
  const int32_t *perm, *bnd, *split_dim;
  const float* thr;
  const uint8_t* lut;
  const float *scale, *offtot;
  uint8_t* codes;
  int64_t* acc;
  float* y;
  int status;
  int summation;        /* 0 exact, 1 avg16 */
} job_t;

static float load_a(const void* A, int dtype, int64_t idx) {
  if (dtype == 0) return ((const float*)A)[idx];
  uint32_t bits = ((uint32_t)((const uint16_t*)A)[idx]) << 16;
  float f;
  memcpy(&f, &bits, sizeof f);
  return f;
}

static void* run_rows(void* arg) {
  job_t* j = (job_t*)arg;
  float* ap = (float*)malloc(sizeof(float) * (size_t)j->D);
  int* code = (int*)malloc(sizeof(int) * (size_t)j->C);
  int64_t* acc = (int64_t*)malloc(sizeof(int64_t) * (size_t)j->M);
  if (!ap || !code || !acc) { j->status = 1; free(ap); free(code); free(acc); return NULL; }
  for (int64_t r = j->r0; r < j->r1; ++r) {
    /* (1) permute the row */
    for (int i = 0; i < j->D; ++i) ap[i] = load_a(j->A, j->dtype, r * j->lda + j->perm[i]);
    /* (2) encode every subspace with its tree */
    for (int c = 0; c < j->C; ++c) {
      const float* chunk = ap + j->bnd[c];
      int node = 0;
      for (int t = 0; t < 4; ++t) {
        float v = chunk[j->split_dim[c * 4 + t]];
        float th = j->thr[c * 15 + ((1 << t) - 1) + node];
        node = 2 * node + (v > th ? 1 : 0);
      }
      code[c] = node;
      if (j->codes) j->codes[r * j->C + c] = (uint8_t)node;
    }
    /* (3) sum of the looked-up LUT rows */
    for (int m = 0; m < j->M; ++m) acc[m] = 0;
    if (j->summation == 0) {
      for (int c = 0; c < j->C; ++c) {
        const uint8_t* row = j->lut + ((int64_t)c * 16 + code[c]) * j->M;
        for (int m = 0; m < j->M; ++m) acc[m] += row[m];
      }
    } else {
      /* (3') groups of 16 codebooks, 4-level rounding-average tree per output, exact group sum */
      for (int g = 0; g < j->C / 16; ++g)
        for (int m = 0; m < j->M; ++m) {
          unsigned v[16];
          for (int i = 0; i < 16; ++i) {
            const int cb = 16 * g + i;
            v[i] = j->lut[((int64_t)cb * 16 + code[cb]) * j->M + m];
          }
          for (int n = 16; n > 1; n /= 2)
            for (int i = 0; i < n / 2; ++i) v[i] = (v[2 * i] + v[2 * i + 1] + 1) >> 1;
          acc[m] += v[0];
        }
    }
    /* (4) dequantise (+ReLU) */
    for (int m = 0; m < j->M; ++m) {
      if (acc[m] >= ((int64_t)1 << 24)) j->status = 2; /* (float)acc must be exact */
      if (j->acc) j->acc[r * j->M + m] = acc[m];
      if (j->y) {
        float yv = j->summation == 0 ? fmaf(j->scale[m], (float)acc[m], j->offtot[m])
                                     : fmaf(16.0f * j->scale[m], (float)acc[m], j->offtot[m]);
        if (j->relu) yv = (yv > 0.0f) ? yv : 0.0f;
        j->y[r * j->M + m] = yv;
      }
    }
  }
  free(ap); free(code); free(acc);
  return NULL;
}

/* Returns 0 on success, 1 on allocation failure, 2 if an accumulator reached 2^24,
 * 3 on invalid arguments.  codes: [N][C] unpacked (one code per byte) or NULL;
 * acc: [N][M] int64 or NULL; y: [N][M] fp32 or NULL.  dtype 0 = fp32, 1 = bf16 bits. */
int oracle_amm2(int64_t N, int D, int C, int M, const void* A, int dtype, int64_t lda,
                const int32_t* perm, const int32_t* bnd, const int32_t* split_dim,
                const float* thr, const uint8_t* lut, const float* scale, const float* offset,
                const float* bias, int relu, uint8_t* codes, int64_t* acc, float* y,
                int nthreads, int summation) {
  if (N < 0 || D < 1 || C < 1 || C > D || M < 1 || lda < D || (dtype != 0 && dtype != 1)) return 3;
  if (summation != 0 && (summation != 1 || C % 16 != 0)) return 3;
  if (N == 0) return 0;
  float* offtot = (float*)malloc(sizeof(float) * (size_t)M);
  if (!offtot) return 1;
  for (int m = 0; m < M; ++m)
    offtot[m] = summation == 0
        ? (float)((double)C * (double)offset[m] + (double)(bias ? bias[m] : 0.0f))
        : (float)((double)C * (double)offset[m] + (double)(bias ? bias[m] : 0.0f) - 16.0 * (C / 16) * (double)scale[m]);
  if (nthreads < 1) nthreads = 1;
  if ((int64_t)nthreads > N) nthreads = (int)N;
  job_t* jobs = (job_t*)calloc((size_t)nthreads, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  if (!jobs || !th) { free(offtot); free(jobs); free(th); return 1; }
  for (int i = 0; i < nthreads; ++i) {
    job_t* j = &jobs[i];
    j->r0 = N * i / nthreads; j->r1 = N * (i + 1) / nthreads;
    j->D = D; j->C = C; j->M = M; j->dtype = dtype; j->relu = relu;
    j->A = A; j->lda = lda; j->perm = perm; j->bnd = bnd; j->split_dim = split_dim;
    j->thr = thr; j->lut = lut; j->scale = scale; j->offtot = offtot;
    j->codes = codes; j->acc = acc; j->y = y; j->status = 0; j->summation = summation;
  }
  int st = 0;
  if (nthreads == 1) {
    run_rows(&jobs[0]);
  } else {
    for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, run_rows, &jobs[i]);
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  }
  for (int i = 0; i < nthreads; ++i) if (jobs[i].status) st = jobs[i].status;
  free(offtot); free(jobs); free(th);
  return st;
}

int oracle_amm(int64_t N, int D, int C, int M, const void* A, int dtype, int64_t lda,
               const int32_t* perm, const int32_t* bnd, const int32_t* split_dim,
               const float* thr, const uint8_t* lut, const float* scale, const float* offset,
               const float* bias, int relu, uint8_t* codes, int64_t* acc, float* y,
               int nthreads) {
  return oracle_amm2(N, D, C, M, A, dtype, lda, perm, bnd, split_dim, thr, lut, scale, offset, bias,
                     relu, codes, acc, y, nthreads, 0);
}
