// tc.cuh — tcgen05 one-hot x LUT tensor-core path.  Placeholder until the
// kernel lands: the plan reports the path as unsupported, AUTO selects SIMT.
#pragma once
#include <vector>
#include "common.cuh"
#include "../../include/itlumm.h"

namespace itlumm {

struct TcPlan {
  bool ok = false;
  const char* why = "tcgen05 path not built";
  const uint8_t* qt = nullptr;
};

struct TcArgs {
  const void* A; int64_t lda; const uint8_t* codes; int64_t ldc; int64_t N;
  int32_t* acc; int64_t ldacc; float* out; int64_t ldo; int relu;
};

inline const char* tc_last_msg() { return "tcgen05 path not built"; }
inline void tc_layout_host(int, int, const uint8_t*, TcPlan*, std::vector<uint8_t>& qt) { qt.clear(); }
inline itlumm_status tc_configure(TcPlan&, int) { return ITLUMM_OK; }
inline bool tc_preferred(const TcPlan& t, bool) { return false && t.ok; }
inline itlumm_status tc_launch(const TcPlan&, const DevPlan&, bool, bool, const TcArgs&, cudaStream_t) {
  return ITLUMM_EUNSUPPORTED;
}

}  // namespace itlumm
