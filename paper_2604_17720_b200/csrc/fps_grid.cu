// K1g instances: binary32 arithmetic, float coordinates (FFPS_F32).
// The kernel (fps_grid.cuh) restates run_kernel, reference
// pkg/src/flashfps/fps_core.py:110-175, with multi-winner rounds.
#include "fps_grid.cuh"

namespace ffps {

const GridInst* grid_instances_f32(int* count) {
  static const GridInst insts[] = {
      FFPS_GRID_PPL(float, float, 8, 1), FFPS_GRID_PPL(float, float, 8, 2), FFPS_GRID_PPL(float, float, 8, 4),
      FFPS_GRID_PPL(float, float, 16, 1), FFPS_GRID_PPL(float, float, 16, 2), FFPS_GRID_PPL(float, float, 16, 4),
  };
  *count = (int)(sizeof(insts) / sizeof(insts[0]));
  return insts;
}

const GridInst* grid_instances(int* count) {
  static GridInst all[128];
  static int n = 0;
  static bool done = false;
  if (!done) {  // first call happens under the C ABI's plan (single-threaded init)
    for (auto get : {grid_instances_f32, grid_instances_f64, grid_instances_mixed}) {
      int c = 0;
      const GridInst* g = get(&c);
      for (int i = 0; i < c && n < 128; ++i) all[n++] = g[i];
    }
    done = true;
  }
  *count = n;
  return all;
}

size_t grid_smem(int dtype, int64_t nb) {
  return dtype == 0 ? grid_smem_bytes<float>(nb)
                    : (dtype == 2 ? grid_smem_bytes<double, float>(nb) : grid_smem_bytes<double>(nb));
}

}  // namespace ffps
