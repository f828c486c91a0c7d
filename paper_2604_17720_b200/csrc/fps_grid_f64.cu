// K1g instances: binary64 arithmetic, double coordinates (FFPS_F64).
// The kernel (fps_grid.cuh) restates run_kernel, reference
// pkg/src/flashfps/fps_core.py:110-175, with multi-winner rounds.
#include "fps_grid.cuh"

namespace ffps {

const GridInst* grid_instances_f64(int* count) {
  static const GridInst insts[] = {
      FFPS_GRID_PPL(double, double, 8, 1), FFPS_GRID_PPL(double, double, 8, 2), FFPS_GRID_PPL(double, double, 8, 4),
      FFPS_GRID_PPL(double, double, 16, 1), FFPS_GRID_PPL(double, double, 16, 2), FFPS_GRID_PPL(double, double, 16, 4),
  };
  *count = (int)(sizeof(insts) / sizeof(insts[0]));
  return insts;
}

}  // namespace ffps
