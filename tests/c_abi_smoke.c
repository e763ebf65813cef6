/* Compiles against include/itlumm.h as plain C99 and links libitlumm.so: every declared entry
 * point is referenced (taking its address) and the ABI version is checked without a GPU.  With a
 * GPU it also pushes data through a plan from C: plan_create -> amm_host -> compare with values
 * worked by hand, and a 1-layer MLP through mlp_forward_host.
 *
 * The hand-worked layer (D = 4, C = 1, M = 2, identity permutation, one 4-dim chunk):
 *   split dims 0,1,2,3 and every threshold 0.5 -> code = 8[x0>.5] + 4[x1>.5] + 2[x2>.5] + [x3>.5]
 *   (reading R1); lut[0][k][m] = k + 16 m, so acc[m] = code + 16 m (a3);
 *   scale = {1, 0.5}, offset = {0, 1}, bias = NULL -> offtot = {0, 1} (R8);
 *   y = fmaf(scale, acc, offtot): row (1,0,1,1) -> code 11 -> {11, 14.5}; row 0 -> {0, 9};
 *   row (1,1,1,1) -> code 15 -> {15, 16.5}; all exact in fp32.  Prints "ok <abi> gpu" or "ok <abi> nogpu". */
#include <stdio.h>
#include <string.h>
#include "itlumm.h"

int main(void) {
  void* fns[] = {(void*)itlumm_plan_create, (void*)itlumm_plan_destroy, (void*)itlumm_plan_set_algo,
                 (void*)itlumm_plan_set_summation, (void*)itlumm_plan_set_onehot, (void*)itlumm_plan_info, (void*)itlumm_encode,
                 (void*)itlumm_lut_accumulate, (void*)itlumm_amm, (void*)itlumm_amm_host,
                 (void*)itlumm_mlp_create, (void*)itlumm_mlp_destroy, (void*)itlumm_mlp_info,
                 (void*)itlumm_mlp_forward, (void*)itlumm_mlp_forward_host, (void*)itlumm_last_launch_count, (void*)itlumm_last_error,
                 (void*)itlumm_abi_version};
  for (unsigned i = 0; i < sizeof fns / sizeof fns[0]; ++i)
    if (!fns[i]) return 2;
  if (itlumm_abi_version() != ITLUMM_ABI_VERSION) return 3;
  if (itlumm_plan_destroy(NULL) != ITLUMM_OK) return 4;
  if (itlumm_amm(NULL, NULL, ITLUMM_F32, 1, 1, NULL, 1, ITLUMM_EPI_NONE, NULL) != ITLUMM_EINVAL) return 5;

  int32_t split_dim[4] = {0, 1, 2, 3};
  float thr[15];
  for (int i = 0; i < 15; ++i) thr[i] = 0.5f;
  uint8_t lut[16 * 2];
  for (int k = 0; k < 16; ++k) { lut[2 * k] = (uint8_t)k; lut[2 * k + 1] = (uint8_t)(k + 16); }
  float scale[2] = {1.0f, 0.5f}, offset[2] = {0.0f, 1.0f};
  itlumm_params p;
  memset(&p, 0, sizeof p);
  p.D = 4; p.C = 1; p.M = 2;
  p.split_dim = split_dim; p.thresholds = thr; p.lut = lut; p.scale = scale; p.offset = offset;
  itlumm_plan plan = NULL;
  if (itlumm_plan_create(&p, 0, &plan) != ITLUMM_OK) {   /* no CUDA device here */
    printf("ok %d nogpu\n", itlumm_abi_version());
    return 0;
  }
  const float A[3][4] = {{1, 0, 1, 1}, {0, 0, 0, 0}, {1, 1, 1, 1}};
  const float want[3][2] = {{11.0f, 14.5f}, {0.0f, 9.0f}, {15.0f, 16.5f}};
  float y[3][2];
  memset(y, 0, sizeof y);
  if (itlumm_amm_host(plan, A, ITLUMM_F32, 4, 3, &y[0][0], 2, ITLUMM_EPI_NONE, NULL) != ITLUMM_OK) {
    fprintf(stderr, "amm_host: %s\n", itlumm_last_error());
    return 6;
  }
  for (int r = 0; r < 3; ++r)
    for (int m = 0; m < 2; ++m)
      if (y[r][m] != want[r][m]) { fprintf(stderr, "amm_host row %d col %d: %g != %g\n", r, m, y[r][m], want[r][m]); return 7; }
  if (itlumm_amm_host(plan, A, ITLUMM_F32, 3, 3, &y[0][0], 2, ITLUMM_EPI_NONE, NULL) != ITLUMM_ESHAPE) return 8;
  itlumm_plan_destroy(plan);

  itlumm_epilogue epi = ITLUMM_EPI_NONE;
  itlumm_mlp mlp = NULL;
  if (itlumm_mlp_create(&p, &epi, 1, 0, &mlp) != ITLUMM_OK) { fprintf(stderr, "mlp_create: %s\n", itlumm_last_error()); return 9; }
  memset(y, 0, sizeof y);
  if (itlumm_mlp_forward_host(mlp, A, ITLUMM_F32, 4, 3, &y[0][0], 2, NULL) != ITLUMM_OK) {
    fprintf(stderr, "mlp_forward_host: %s\n", itlumm_last_error());
    return 10;
  }
  for (int r = 0; r < 3; ++r)
    for (int m = 0; m < 2; ++m)
      if (y[r][m] != want[r][m]) { fprintf(stderr, "mlp row %d col %d: %g != %g\n", r, m, y[r][m], want[r][m]); return 11; }
  itlumm_mlp_destroy(mlp);
  printf("ok %d gpu\n", itlumm_abi_version());
  return 0;
}
