/* itlumm.h — C ABI of the B200-native ITLUMM / MADDNESS inference hot path.
 *
 * The problem: approximate sigma(A.B) for a FIXED weight
 * matrix B that has been folded offline into a lookup table h(B) = quantise(P.B), with a learned
 * encoder g(A).  Per activation row a:
 *   a1  permutation / partition: a'[i] = a[perm[i]], chunk c = a'[b_c .. b_{c+1})
 *   a2  encode: depth-4 balanced regression tree, K = 16, "exactly 4 comparisons":
 *         node = 0; for t = 0..3: node = 2*node + (chunk_c[split_dim[c][t]] > thr[c][2^t-1+node])
 *         code_c = node
 *   a3  lookup-accumulate: acc[m] = sum_c lut[c][code_c][m], uint8 entries summed EXACTLY in
 *         32-bit integers ("rounded 8-bit summation": reading R7 in DESIGN.md)
 *   a4  dequantise (+ReLU): y[m] = fmaf(scale[m], (float)acc[m], offtot[m]) with
 *         offtot[m] = (float)((double)C*(double)offset[m] + (double)bias[m])     (reading R8);
 *         ReLU: y > 0 ? y : +0                                                     (R9)
 * K = 16 is fixed.  Every entry point is asynchronous on `stream` unless stated otherwise.
 *
 * Conventions for every call
 *   - Status codes: ITLUMM_OK on success; otherwise the call has no effect on outputs and
 *     itlumm_last_error() returns a thread-local message naming the failed check.
 *   - Device pointers are caller-owned CUDA device allocations on the plan's device; host
 *     pointers are caller-owned host memory.  The library never frees caller memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - N = 0 returns ITLUMM_OK without launching anything.
 *   - There is NO CPU fallback: a kernel that cannot run returns ITLUMM_EUNSUPPORTED/ECUDA.
 *   - Asynchronous device faults surface at the caller's next synchronisation.
 *   - Concurrent calls on one plan from several host threads/streams are safe: the plan is
 *     immutable after creation ("pure and reentrant"), except itlumm_amm_host, which
 *     uses plan-owned staging buffers and serialises itself with a mutex.
 */
#ifndef ITLUMM_H
#define ITLUMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ITLUMM_ABI_VERSION 5

typedef enum {
  ITLUMM_OK = 0,
  ITLUMM_EINVAL = 1,        /* bad argument: null pointer, bad size/stride, invalid parameters */
  ITLUMM_ESHAPE = 2,        /* call inconsistent with the plan's dims ("shape
                               mismatch"): lda < D, ldc < ceil(C/2), ldo or ldacc < M, or an MLP
                               whose layer l+1 has D != M of layer l                           */
  ITLUMM_EUNSUPPORTED = 3,  /* shape/dtype/alignment the selected kernel cannot take          */
  ITLUMM_ECUDA = 4,         /* CUDA launch/config/runtime failure (cudaGetErrorString in msg) */
  ITLUMM_ENOMEM = 5         /* device or host allocation failure                             */
} itlumm_status;

typedef enum { ITLUMM_F32 = 0, ITLUMM_BF16 = 1 } itlumm_dtype;            /* element type of A */
typedef enum { ITLUMM_EPI_NONE = 0, ITLUMM_EPI_RELU = 1 } itlumm_epilogue;  /* sigma    */

/* Kernel schedule used by itlumm_amm / itlumm_amm_host / itlumm_lut_accumulate.
 *   AUTO    : library choice: TC_PIPE (itlumm_amm) / TC
 *             (itlumm_lut_accumulate) where the tensor-core tiling applies, else SIMT.  If a
 *             tensor-core kernel cannot take the codes it is given (a streamed LUT needs codes rows
 *             that are 16-byte multiples), itlumm_lut_accumulate runs the SIMT kernel instead.
 *   SIMT    : CUDA-core shared-memory LUT kernels; itlumm_amm = one fused kernel.
 *   TC      : tcgen05 one-hot x LUT int8 tensor-core kernel (G.T with G the one-hot encoding,
 *             P:89; exact integer products); itlumm_amm = one fused kernel (encode inside) where the
 *             LUT stays resident in shared memory.
 *   TC_PIPE : itlumm_amm = the encode kernel writing codes to a plan-owned, L2-resident scratch
 *             buffer, then the TC accumulate kernel (2 launches; concurrent calls on one plan
 *             are serialised on the device through an event).  itlumm_lut_accumulate = TC.
 * Where the LUT is too large to stay resident (it is then streamed K-block by K-block), the TC
 * accumulate runs on CTA pairs (tcgen05.mma.cta_group::2, each SM stages half of every LUT block).
 * TC and TC_PIPE return EUNSUPPORTED where the tensor-core tiling does not apply.  Every
 * schedule produces bit-identical results. */
typedef enum {
  ITLUMM_ALGO_AUTO = 0, ITLUMM_ALGO_SIMT = 1, ITLUMM_ALGO_TC = 2, ITLUMM_ALGO_TC_PIPE = 3
} itlumm_algo;

/* Summation over codebooks (a3).
 *   EXACT : acc[m] = sum_c lut[c][code_c][m], exact in int32 (reading R7; the default).
 *   AVG16 : MADDNESS's "fast rounded 8-bit summation" (reading R22): codebooks in
 *           groups of 16 (C % 16 == 0), per output a 4-level tree of per-byte rounding averages
 *           avg(a,b) = (a+b+1)>>1 over the group's 16 entries (pairs (0,1),(2,3),... per level),
 *           acc[m] = sum of the group results; y = fmaf(16*scale, (float)acc, offavg) with
 *           offavg = (float)((double)C*offset + bias - 16*(C/16)*(double)scale) (the tree's +1
 *           expected bias per group removed).  CUDA-core kernels only. */
typedef enum { ITLUMM_SUM_EXACT = 0, ITLUMM_SUM_AVG16 = 1 } itlumm_summation;

/* Operand form of the one-hot matrix G on the tensor-core paths (TC, TC_PIPE).
 *   AUTO     : library choice: DENSE (measured fastest on every kernel).
 *   DENSE    : G as u8 (16 bytes per codebook), tcgen05.mma kind::i8, K = 32 per instruction.
 *   SPARSE24 : G is 1-of-16 per codebook, hence 2:4 sparse: stored compressed (8 bytes per
 *              codebook) with 2-bit position metadata per stored element, tcgen05.mma.sp kind::i8,
 *              K = 64 per instruction; N slices of at most 224 columns (TMEM holds the metadata).
 * All give the same exact integer products (bit-identical results). */
typedef enum {
  ITLUMM_ONEHOT_AUTO = 0, ITLUMM_ONEHOT_DENSE = 1, ITLUMM_ONEHOT_SPARSE24 = 2
} itlumm_onehot;

typedef struct itlumm_plan_s* itlumm_plan; /* opaque; owns device copies of all parameters */

/* Fitted layer parameters.  HOST pointers, read only during itlumm_plan_create (copied). */
typedef struct {
  int32_t D;                 /* input dim (columns of A)                                     */
  int32_t C;                 /* codebooks, 1 <= C <= D                                      */
  int32_t M;                 /* output dim (columns of B / of the result)                    */
  const int32_t* perm;       /* [D] bijection, a'[i] = a[perm[i]]; NULL = identity (R11)     */
  const int32_t* boundaries; /* [C+1], 0 = b_0 < b_1 < ... < b_C = D; NULL = equal chunks,
                                larger first (R12: first D mod C chunks get one extra dim)  */
  const int32_t* split_dim;  /* [C][4] subspace-local split dim per level, 0 <= sd < d_c     */
  const float* thresholds;   /* [C][15] heap order: level t, node n at (2^t - 1) + n; no NaN
                                (+-inf allowed)                                  */
  const uint8_t* lut;        /* [C][16][M] quantised table q (16*C*M bytes)            */
  const float* scale;        /* [M] per-output scale, finite                                 */
  const float* offset;       /* [M] per-output offset lo_m (min of column m of T), finite    */
  const float* bias;         /* [M] or NULL (= 0), finite                                     */
} itlumm_params;

/* Validate `p`, fold the permutation into absolute gather columns
 * col[c][t] = perm[b_c + split_dim[c][t]], compute offtot, lay the LUT out for the kernels and
 * copy everything to `cuda_device`.  Blocking.  On success *out owns the device copies.
 * Errors: EINVAL (null required pointer; D, C or M < 1; C > D; perm not a bijection;
 * boundaries not strictly increasing from 0 to D; split_dim outside [0, d_c); NaN threshold;
 * non-finite scale/offset/bias; bad device), ENOMEM, ECUDA. */
itlumm_status itlumm_plan_create(const itlumm_params* p, int cuda_device, itlumm_plan* out);

/* Free the plan's device memory (synchronises the plan's device).  NULL is a no-op. */
itlumm_status itlumm_plan_destroy(itlumm_plan plan);

/* Select the kernel family (default AUTO).  Not thread-safe against concurrent launches. */
itlumm_status itlumm_plan_set_algo(itlumm_plan plan, itlumm_algo algo);

/* Select the summation (default EXACT).  AVG16 needs C % 16 == 0 (else EINVAL) and runs on the
 * CUDA-core kernels whatever the algo (acc outputs are then the group-average sums).  Not
 * thread-safe against concurrent launches. */
itlumm_status itlumm_plan_set_summation(itlumm_plan plan, itlumm_summation summation);

/* Select the one-hot operand form (default AUTO).  EUNSUPPORTED when the tensor-core tiling of
 * that form does not apply to the plan.  Not thread-safe against concurrent launches. */
itlumm_status itlumm_plan_set_onehot(itlumm_plan plan, itlumm_onehot onehot);

/* Query plan dims: any out-pointer may be NULL.  lut_bytes = 16*C*M. */
itlumm_status itlumm_plan_info(itlumm_plan plan, int32_t* D, int32_t* C, int32_t* M,
                               int64_t* lut_bytes);

/* a1 + a2.  A: device, N rows x lda elements of `dtype`, row-major, lda >= D; only the 4C
 * split columns of each row are read.  codes: device, N x ldc bytes, ldc >= ceil(C/2);
 * row r byte i holds code 2i in its low nibble and code 2i+1 in its high nibble (R14; an odd
 * C leaves the last high nibble 0).  Errors: EINVAL (null, N < 0, bad dtype, A or codes not device
 * memory of the plan's device), ESHAPE (lda < D, ldc < ceil(C/2)), ECUDA. */
itlumm_status itlumm_encode(itlumm_plan plan, const void* A, itlumm_dtype dtype, int64_t lda,
                            int64_t N, uint8_t* codes, int64_t ldc, void* stream);

/* a3 (+ a4).  codes as produced by itlumm_encode.  acc: device int32 [N][ldacc] (ldacc >= M)
 * or NULL; out: device fp32 [N][ldo] (ldo >= M) or NULL; at least one must be non-NULL.
 * `epi` applies to `out` only.  Errors: EINVAL (null codes, both outputs NULL, a pointer that is
 * not device memory of the plan's device), ESHAPE (ldc < ceil(C/2), ldacc or ldo < M),
 * EUNSUPPORTED, ECUDA. */
itlumm_status itlumm_lut_accumulate(itlumm_plan plan, const uint8_t* codes, int64_t ldc,
                                    int64_t N, int32_t* acc, int64_t ldacc, float* out,
                                    int64_t ldo, itlumm_epilogue epi, void* stream);

/* a1..a4 in one call.  With SIMT/TC one fused kernel (codes never leave the SM); with
 * TC_PIPE (AUTO's choice when M is split across CTAs) encode + accumulate kernels exchanging
 * the codes (ceil(C/2) bytes per row) through an L2-resident scratch buffer.  A as in
 * itlumm_encode, out device fp32 [N][ldo], ldo >= M.  Errors: EINVAL (null, N < 0, bad dtype, A or
 * out not device memory of the plan's device), ESHAPE (lda < D, ldo < M), EUNSUPPORTED, ECUDA. */
itlumm_status itlumm_amm(itlumm_plan plan, const void* A, itlumm_dtype dtype, int64_t lda,
                         int64_t N, float* out, int64_t ldo, itlumm_epilogue epi, void* stream);

/* Fused a1..a4 on HOST buffers (end-to-end API).  A_host: N x lda elements (pinned memory is
 * fastest; pageable works), out_host: N x ldo fp32.  Rows are streamed through plan-owned
 * device staging buffers in chunks with H2D copy / kernel / D2H copy overlapped across three
 * internal streams.  Ordered after prior work on `stream`; BLOCKING: returns when out_host is
 * written.  Staging is allocated on first use (ENOMEM possible) and kept by the plan.
 * Errors: as itlumm_amm, plus ENOMEM. */
itlumm_status itlumm_amm_host(itlumm_plan plan, const void* A_host, itlumm_dtype dtype,
                              int64_t lda, int64_t N, float* out_host, int64_t ldo,
                              itlumm_epilogue epi, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Whole-network chaining (BASELINE configs[3]: every linear layer of an MLP
 * replaced by ITLUMM).  Layer l+1 consumes layer l's fp32 output.  Because a layer's
 * encoder reads only its 4C split columns, layer l computes ONLY the (sorted, distinct) output
 * columns layer l+1 splits on, into a compacted device buffer that layer l+1 reads through a
 * re-mapped gather ("dead-column elimination"); the last layer computes all its columns.  The
 * final outputs are bit-identical to running every layer in full (same LUT columns, same fmaf).
 * --------------------------------------------------------------------------------------------- */
typedef struct itlumm_mlp_s* itlumm_mlp; /* opaque; owns one plan per layer + intermediate buffers */

/* layers[l]: host params as for itlumm_plan_create (read during the call only); requires
 * layers[l+1].D == layers[l].M.  epis[l]: sigma of layer l (ReLU on hidden layers).
 * Errors: as itlumm_plan_create (message prefixed with the layer index), ESHAPE on a shape chain
 * mismatch, EINVAL on n_layers < 1. */
itlumm_status itlumm_mlp_create(const itlumm_params* layers, const itlumm_epilogue* epis,
                                int32_t n_layers, int cuda_device, itlumm_mlp* out);

/* Free the layers' plans and buffers (synchronises the device).  NULL is a no-op. */
itlumm_status itlumm_mlp_destroy(itlumm_mlp mlp);

/* widths[l] (host, n_layers entries, may be NULL) = output columns layer l computes. */
itlumm_status itlumm_mlp_info(itlumm_mlp mlp, int32_t* n_layers, int32_t* widths);

/* Forward pass: A device [N][lda] (dtype; lda >= layers[0].D) -> out device fp32 [N][ldo]
 * (ldo >= last layer's M).  Rows are processed in chunks of up to 262144 through plan-owned
 * intermediate buffers (allocated on first use: ENOMEM possible).  Async on `stream`; calls on one
 * MLP are serialised on the device by the stream order the caller gives them.
 * Errors: EINVAL, ESHAPE (lda < layers[0].D, ldo < last M), ENOMEM, EUNSUPPORTED, ECUDA. */
itlumm_status itlumm_mlp_forward(itlumm_mlp mlp, const void* A, itlumm_dtype dtype, int64_t lda,
                                 int64_t N, float* out, int64_t ldo, void* stream);

/* Forward pass on HOST buffers (end-to-end API, as itlumm_amm_host): A_host [N][lda] (dtype),
 * out_host fp32 [N][ldo].  Rows stream through MLP-owned device staging in ~64 MB chunks; the H2D
 * of chunk i+1 and the D2H of chunk i-1 overlap the forward of chunk i (forwards run on `stream`).
 * BLOCKING: returns when out_host is written.  Errors: as itlumm_mlp_forward. */
itlumm_status itlumm_mlp_forward_host(itlumm_mlp mlp, const void* A_host, itlumm_dtype dtype, int64_t lda,
                                      int64_t N, float* out_host, int64_t ldo, void* stream);

/* Number of kernel launches the last successful launching call on this thread made. */
int32_t itlumm_last_launch_count(void);

/* Thread-local message for the last non-OK status on this thread ("" if none). */
const char* itlumm_last_error(void);

/* ITLUMM_ABI_VERSION of the loaded library. */
int32_t itlumm_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ITLUMM_H */
