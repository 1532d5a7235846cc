// psso_registry.h -- lookup of the k_tile template instantiations, which are
// compiled in separate translation units (psso_tiles_*.cu) to build in parallel.
#pragma once

namespace psso {
const void* tile_kernel_f64_ref(int fn, int vec);
const void* tile_kernel_f64_philox(int fn, int vec);
const void* tile_kernel_f32_ref(int fn, int vec);
const void* tile_kernel_f32_philox(int fn, int vec);

inline const void* tile_kernel(int dtype, int rng, int fn, int vec) {
  if (dtype == 0) return rng == 0 ? tile_kernel_f64_ref(fn, vec) : tile_kernel_f64_philox(fn, vec);
  return rng == 0 ? tile_kernel_f32_ref(fn, vec) : tile_kernel_f32_philox(fn, vec);
}
}  // namespace psso
