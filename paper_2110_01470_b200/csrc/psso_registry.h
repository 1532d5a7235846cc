// psso_registry.h -- lookup of the k_tile template instantiations, which are
// compiled in separate translation units (psso_tiles_*.cu) to build in parallel.
#pragma once

namespace psso {
const void* tile_kernel_f64_ref(int fn, int vec, bool fused);
const void* tile_kernel_f64_philox(int fn, int vec, bool fused);
const void* tile_kernel_f32_ref(int fn, int vec, bool fused);
const void* tile_kernel_f32_philox(int fn, int vec, bool fused);

const void* chain_kernel_f64_ref(int fn, int m, bool init);
const void* chain_kernel_f64_philox(int fn, int m, bool init);
const void* chain_kernel_f32_ref(int fn, int m, bool init);
const void* chain_kernel_f32_philox(int fn, int m, bool init);

inline const void* chain_kernel(int dtype, int rng, int fn, int m, bool init) {
  if (dtype == 0)
    return rng == 0 ? chain_kernel_f64_ref(fn, m, init) : chain_kernel_f64_philox(fn, m, init);
  return rng == 0 ? chain_kernel_f32_ref(fn, m, init) : chain_kernel_f32_philox(fn, m, init);
}

inline const void* tile_kernel(int dtype, int rng, int fn, int vec, bool fused) {
  if (dtype == 0)
    return rng == 0 ? tile_kernel_f64_ref(fn, vec, fused) : tile_kernel_f64_philox(fn, vec, fused);
  return rng == 0 ? tile_kernel_f32_ref(fn, vec, fused) : tile_kernel_f32_philox(fn, vec, fused);
}
}  // namespace psso
