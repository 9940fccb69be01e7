// k_fused instantiations of the count-free path (k_prep before it instead of
// k_count; every row short by construction): kShortRowsPerTile rows per warp
// tile, like fused_short.cu, with the count-free checks compiled in; and for
// small products the same with the prep pass inside (PREP 1 / 2).
#include "fused_launch.cuh"

namespace spmmm {
cudaError_t fused_cf(int op, const FusedParams& prm, const FusedLaunchEnv& env, bool wide,
                     bool stats, unsigned grid, int* occ, int prep) {
  if (prep == 1)
    return fused_dispatch<kFusedWarps, kShortRowsPerTile, false, true, 1>(op, prm, env, wide,
                                                                          stats, grid, occ);
  if (prep == 2)
    return fused_dispatch<kFusedWarps, kShortRowsPerTile, false, true, 2>(op, prm, env, wide,
                                                                          stats, grid, occ);
  return fused_dispatch<kFusedWarps, kShortRowsPerTile, false, true, 0>(op, prm, env, wide, stats,
                                                                        grid, occ);
}
}  // namespace spmmm
