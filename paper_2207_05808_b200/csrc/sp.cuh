// sp.cuh — spatially partitioned persistent pipeline: the fused itlumm_amm in ONE launch.
//
// The two halves of the path have different bottlenecks: a1+a2 (encode) streams whole rows of A
// in (the split columns are scattered, so DRAM fetches ~every line), a3'+a4 (one-hot x LUT on
// tcgen05 + dequant) streams the fp32 output out.  Run back to back (TC_PIPE) each kernel pays
// its own fill and tail, and HBM reads and writes never overlap.  Here one cooperative grid of one
// CTA per SM is split: the first E CTAs run the encoder (enc_cta: TMA row ring -> codes into an
// L2-resident buffer), the other T CTAs run the tensor-core accumulator (tc_cta, G slices of M).
// Codes flow through L2: after its share of an encode tile each encoder warp fences and bumps the
// ready counter of the 128-row TC tile; the TC loader warp waits on that counter before the bulk
// copy of the tile's codes.  Encoders never wait on the TC side and the codes buffer holds every
// row of the call, so there is no cycle; the cooperative launch guarantees co-residency.
#pragma once
#include "encode.cuh"
#include "tc.cuh"

namespace itlumm {

struct SpArgs {
  int E;    // encoder CTAs (blockIdx < E); the remaining CTAs (a multiple of G) run tc_cta
};

template <typename T, bool SB>
__global__ void __launch_bounds__(kTcThreads, 1) k_amm_sp(DevPlan p, EncArgs ge, TcKArgs gt, SpArgs sp,
                                                         const __grid_constant__ CUtensorMap out_map) {
  extern __shared__ __align__(1024) uint8_t smem_sp[];
  if ((int)blockIdx.x < sp.E) {
    if (p.C >= 32) enc_cta<T, true>(p, ge, smem_sp, blockIdx.x, sp.E, gt.ready);
    else enc_cta<T, false>(p, ge, smem_sp, blockIdx.x, sp.E, gt.ready);
  } else {
    tc_cta<false, float, SB>(p, gt, &out_map, smem_sp, blockIdx.x - sp.E, gridDim.x - sp.E);
  }
}

}  // namespace itlumm
