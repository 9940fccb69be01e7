// k_fused instantiations of the count-free path (k_prep before it instead of
// k_count; every row short by construction): kShortRowsPerTile rows per warp
// tile, like fused_short.cu, with the count-free checks compiled in.
#include "fused_launch.cuh"

namespace spmmm {
cudaError_t fused_cf(int op, const FusedParams& prm, const FusedLaunchEnv& env, bool wide,
                     bool stats, unsigned grid, int* occ) {
  return fused_dispatch<kFusedWarps, kShortRowsPerTile, false, true>(op, prm, env, wide, stats,
                                                                     grid, occ);
}
}  // namespace spmmm
