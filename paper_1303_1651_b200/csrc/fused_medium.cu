// k_fused instantiations with per-warp shared-memory tables (medium rows),
// one row per warp tile.
#include "fused_launch.cuh"

namespace spmmm {
cudaError_t fused_medium(int op, const FusedParams& prm, const FusedLaunchEnv& env, bool wide,
                         bool stats, unsigned grid, int* occ) {
  return fused_dispatch<kFusedWarps, 1, true>(op, prm, env, wide, stats, grid, occ);
}
}  // namespace spmmm
