/* Compiles against include/itlumm.h as plain C99 and links libitlumm.so: every declared entry
 * point is referenced (taking its address), and the ABI version is checked without a GPU. */
#include <stdio.h>
#include "itlumm.h"

int main(void) {
  void* fns[] = {(void*)itlumm_plan_create, (void*)itlumm_plan_destroy, (void*)itlumm_plan_set_algo,
                 (void*)itlumm_plan_set_summation, (void*)itlumm_plan_set_onehot, (void*)itlumm_plan_info, (void*)itlumm_encode,
                 (void*)itlumm_lut_accumulate, (void*)itlumm_amm, (void*)itlumm_amm_host,
                 (void*)itlumm_mlp_create, (void*)itlumm_mlp_destroy, (void*)itlumm_mlp_info,
                 (void*)itlumm_mlp_forward, (void*)itlumm_last_launch_count, (void*)itlumm_last_error,
                 (void*)itlumm_abi_version};
  for (unsigned i = 0; i < sizeof fns / sizeof fns[0]; ++i)
    if (!fns[i]) return 2;
  if (itlumm_abi_version() != ITLUMM_ABI_VERSION) return 3;
  if (itlumm_plan_destroy(NULL) != ITLUMM_OK) return 4;
  if (itlumm_amm(NULL, NULL, ITLUMM_F32, 1, 1, NULL, 1, ITLUMM_EPI_NONE, NULL) != ITLUMM_EINVAL) return 5;
  printf("ok %d\n", itlumm_abi_version());
  return 0;
}
