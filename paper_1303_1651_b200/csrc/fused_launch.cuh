// Launch entry points of the fused kernel, one translation unit per shared
// table size (fused_t0.cu ... fused_t1024.cu) so they compile in parallel.
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace spmmm {

constexpr int kFusedWarps = 8;
constexpr int kFusedShortRowsPerWarp = 4;

struct FusedLaunchEnv {
  int device;
  int sms;
  cudaStream_t stream;
};

// Cooperative (all blocks co-resident) persistent launch: grid = min(tiles,
// resident blocks per SM * SMs). The look-back requires co-residency.
template <int WARPS, int R, int T, bool WIDE, bool STATS>
cudaError_t launch_fused(const FusedParams& prm_in, const FusedLaunchEnv& env) {
  auto kern = k_fused<WARPS, R, T, WIDE, STATS>;
  const size_t smem = size_t(WARPS) * size_t(T) * (sizeof(double) + sizeof(uint32_t));
  static int occ_cache[64] = {};
  int& occ = occ_cache[env.device & 63];
  if (occ == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, WARPS * 32, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
  }
  FusedParams prm = prm_in;
  const unsigned long long max_grid = (unsigned long long)occ * (unsigned long long)env.sms;
  const unsigned grid = unsigned(prm.ntiles < max_grid ? prm.ntiles : max_grid);
  void* args[] = {&prm};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(grid), dim3(WARPS * 32),
                                     args, smem, env.stream);
}

template <int WARPS, int R, int T>
cudaError_t launch_fused_kw(const FusedParams& prm, const FusedLaunchEnv& env, bool wide,
                            bool stats) {
  if (wide) return stats ? launch_fused<WARPS, R, T, true, true>(prm, env)
                         : launch_fused<WARPS, R, T, true, false>(prm, env);
  return stats ? launch_fused<WARPS, R, T, false, true>(prm, env)
               : launch_fused<WARPS, R, T, false, false>(prm, env);
}

cudaError_t launch_fused_t0(const FusedParams&, const FusedLaunchEnv&, bool wide, bool stats);
cudaError_t launch_fused_t256(const FusedParams&, const FusedLaunchEnv&, bool wide, bool stats);
cudaError_t launch_fused_t512(const FusedParams&, const FusedLaunchEnv&, bool wide, bool stats);
cudaError_t launch_fused_t1024(const FusedParams&, const FusedLaunchEnv&, bool wide, bool stats);

}  // namespace spmmm
