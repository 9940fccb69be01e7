// k_fused instantiations for split mode (skewed inputs: the non-short rows
// are computed before k_fused by the ESC / long-row kernels): the counted
// short variant with packed passes for groups of tiny rows and without the
// ELL path (kernels.cuh SPLIT).
#include "fused_launch.cuh"

namespace spmmm {
cudaError_t fused_split(int op, const FusedParams& prm, const FusedLaunchEnv& env, bool wide,
                        bool stats, unsigned grid, int* occ) {
  return fused_dispatch<kFusedWarps, kShortRowsPerTile, false, false, 0, true>(op, prm, env, wide,
                                                                               stats, grid, occ);
}
}  // namespace spmmm
