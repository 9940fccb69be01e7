// k_fused instantiations of the count-free path (k_prep before it instead of
// k_count; every row short by construction): kShortRowsPerTile rows per warp
// tile, like fused_short.cu, with the count-free checks compiled in; and for
// small products the same with the prep pass inside (PREP 1 / 2). C = A·A
// (large) runs the instantiations with the self-record path (SELF): kept out
// of the ones A != B products run — compiled into them it cost C3 2.8%.
#include "fused_launch.cuh"

namespace spmmm {
cudaError_t fused_cf(int op, const FusedParams& prm, const FusedLaunchEnv& env, bool wide,
                     bool stats, unsigned grid, int* occ, int prep, bool self) {
  // (the small products of prep 1 are C = A·A too, but launch-bound: the
  // self-record path measured 0.6 us slower on C1, 35.3 against 34.7)
  if (prep == 1)
    return fused_dispatch<kFusedWarps, kShortRowsPerTile, false, true, 1>(op, prm, env, wide,
                                                                          stats, grid, occ);
  if (prep == 2)
    return fused_dispatch<kFusedWarps, kShortRowsPerTile, false, true, 2>(op, prm, env, wide,
                                                                          stats, grid, occ);
  if (self)
    return fused_dispatch<kFusedWarps, kShortRowsPerTile, false, true, 0, false, true>(
        op, prm, env, wide, stats, grid, occ);
  return fused_dispatch<kFusedWarps, kShortRowsPerTile, false, true, 0>(op, prm, env, wide, stats,
                                                                        grid, occ);
}
}  // namespace spmmm
