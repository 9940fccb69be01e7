// k_fused instantiations for products whose rows are all short (<= 32
// products): no tables, kShortRowsPerTile rows per warp tile.
#include "fused_launch.cuh"

namespace spmmm {
cudaError_t fused_short(int op, const FusedParams& prm, const FusedLaunchEnv& env, bool wide,
                        bool stats, unsigned grid, int* occ) {
  return fused_dispatch<kFusedWarps, kShortRowsPerTile, false>(op, prm, env, wide, stats, grid,
                                                               occ);
}
}  // namespace spmmm
