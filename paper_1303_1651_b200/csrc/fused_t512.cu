// k_fused instantiations for a shared-memory table of 512 slots per warp.
#include "fused_launch.cuh"

namespace spmmm {
cudaError_t launch_fused_t512(const FusedParams& prm, const FusedLaunchEnv& env, bool wide,
                            bool stats) {
  return launch_fused_kw<kFusedWarps, 1, 512>(prm, env, wide, stats);
}
}  // namespace spmmm
