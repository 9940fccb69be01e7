// k_fused instantiations for split mode (skewed inputs: the non-short rows
// are computed before k_fused by the ESC / long-row kernels): the counted
// short variant whose tiles go through packed passes only — up to 8 tiny rows
// per expand-sort-fold pass (kernels.cuh SPLIT, rows.cuh packed_tile_pass).
// Used without row stats and for columns < 2^24 (or 64-bit keys); otherwise
// split mode runs the shared short variant.
#include "fused_launch.cuh"

namespace spmmm {
cudaError_t fused_split(int op, const FusedParams& prm, const FusedLaunchEnv& env, bool wide,
                        bool stats, unsigned grid, int* occ) {
  return fused_dispatch<kFusedWarps, kShortRowsPerTile, false, false, 0, true>(op, prm, env, wide,
                                                                               stats, grid, occ);
}
}  // namespace spmmm
