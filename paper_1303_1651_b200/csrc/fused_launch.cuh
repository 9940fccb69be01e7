// Launch entry points of the fused kernel. The short-only and the medium
// variants live in separate translation units (fused_short.cu,
// fused_medium.cu) so they compile in parallel.
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace spmmm {

#ifndef SPMMM_FUSED_WARPS
#define SPMMM_FUSED_WARPS 8
#endif
constexpr int kFusedWarps = SPMMM_FUSED_WARPS;
#ifndef SPMMM_SHORT_BLOCKS
#define SPMMM_SHORT_BLOCKS 4  // resident blocks per SM the short variant is compiled for
#endif
#ifndef SPMMM_SHORT_ROWS
#define SPMMM_SHORT_ROWS 8
#endif
constexpr int kShortRowsPerTile = SPMMM_SHORT_ROWS;  // rows per warp tile without medium rows

struct FusedLaunchEnv {
  int device;
  int sms;
  cudaStream_t stream;
};

template <int WARPS, int R, bool MEDIUM, bool WIDE, bool STATS, bool CF = false, int PREP = 0,
          bool SPLIT = false, bool SELF = false>
struct FusedVariant {
  static constexpr size_t smem() {
    return FusedSmem<R, MEDIUM>::bytes(WARPS);
  }
  // resident blocks per SM (cached per device)
  static cudaError_t occupancy(int device, int* occ) {
    static int cache[64] = {};
    int& c = cache[device & 63];
    if (c == 0) {
      auto kern = k_fused<WARPS, R, MEDIUM, WIDE, STATS, CF, PREP, SPLIT, SELF>;
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           int(smem()));
      if (e != cudaSuccess) return e;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, kern, WARPS * 32, smem());
      if (e != cudaSuccess) return e;
      if (c < 1) return cudaErrorInvalidConfiguration;
    }
    *occ = c;
    return cudaSuccess;
  }
  // cooperative launch: the look-back needs every warp co-resident
  static cudaError_t launch(const FusedParams& prm_in, const FusedLaunchEnv& env, unsigned grid) {
    FusedParams prm = prm_in;
    void* args[] = {&prm};
    return cudaLaunchCooperativeKernel(
        reinterpret_cast<void*>(k_fused<WARPS, R, MEDIUM, WIDE, STATS, CF, PREP, SPLIT, SELF>), dim3(grid),
        dim3(WARPS * 32), args, smem(), env.stream);
  }
};

// op 0: occupancy query into *occ; op 1: launch with `grid`
cudaError_t fused_short(int op, const FusedParams& prm, const FusedLaunchEnv& env, bool wide,
                        bool stats, unsigned grid, int* occ);
// the split-mode short variant (fused_split.cu): packed passes, no ELL path
cudaError_t fused_split(int op, const FusedParams& prm, const FusedLaunchEnv& env, bool wide,
                        bool stats, unsigned grid, int* occ);
cudaError_t fused_medium(int op, const FusedParams& prm, const FusedLaunchEnv& env, bool wide,
                         bool stats, unsigned grid, int* occ);
// the count-free short variant (fused_cf.cu); prep 1 / 2: with the prep pass
// of mode 0 / 1 inside (small products)
// self: C = A·A (the instantiations with the self-record path compiled in)
cudaError_t fused_cf(int op, const FusedParams& prm, const FusedLaunchEnv& env, bool wide,
                     bool stats, unsigned grid, int* occ, int prep, bool self);

template <int WARPS, int R, bool MEDIUM, bool CF = false, int PREP = 0, bool SPLIT = false,
          bool SELF = false>
cudaError_t fused_dispatch(int op, const FusedParams& prm, const FusedLaunchEnv& env, bool wide,
                           bool stats, unsigned grid, int* occ) {
#define SPMMM_FUSED_CASE(W, S)                                                  \
  if (wide == W && stats == S) {                                                \
    using V = FusedVariant<WARPS, R, MEDIUM, W, S, CF, PREP, SPLIT, SELF>;                   \
    return op == 0 ? V::occupancy(env.device, occ) : V::launch(prm, env, grid); \
  }
  SPMMM_FUSED_CASE(false, false)
  SPMMM_FUSED_CASE(false, true)
  SPMMM_FUSED_CASE(true, false)
  SPMMM_FUSED_CASE(true, true)
#undef SPMMM_FUSED_CASE
  return cudaErrorInvalidValue;
}

}  // namespace spmmm
