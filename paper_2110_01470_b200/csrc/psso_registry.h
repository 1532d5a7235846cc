// psso_registry.h -- lookup of the k_tile / k_fused / k_chain template instantiations, which are
// compiled in separate translation units (psso_tiles_*.cu) to build in parallel.
#pragma once

namespace psso {
const void* tile_kernel_f64_ref(int fn, int vec, bool fused);
const void* tile_kernel_f64_philox(int fn, int vec, bool fused);
const void* tile_kernel_f32_ref(int fn, int vec, bool fused);
const void* tile_kernel_f32_philox(int fn, int vec, bool fused);

const void* chain_kernel_f64_ref(int fn, int m, bool init, bool full);
const void* chain_kernel_f64_philox(int fn, int m, bool init, bool full);
const void* chain_kernel_f32_ref(int fn, int m, bool init, bool full);
const void* chain_kernel_f32_philox(int fn, int m, bool init, bool full);

const void* rows_kernel_f64_ref(int fn, int w);
const void* rows_kernel_f64_philox(int fn, int w);
const void* rows_kernel_f32_ref(int fn, int w);
const void* rows_kernel_f32_philox(int fn, int w);

inline const void* rows_kernel(int dtype, int rng, int fn, int w) {
  if (dtype == 0) return rng == 0 ? rows_kernel_f64_ref(fn, w) : rows_kernel_f64_philox(fn, w);
  return rng == 0 ? rows_kernel_f32_ref(fn, w) : rows_kernel_f32_philox(fn, w);
}

const void* swarm_kernel_f64_ref(int fn, int m, bool res, bool cl);
const void* swarm_kernel_f64_philox(int fn, int m, bool res, bool cl);
const void* swarm_kernel_f32_ref(int fn, int m, bool res, bool cl);
const void* swarm_kernel_f32_philox(int fn, int m, bool res, bool cl);

inline const void* swarm_kernel(int dtype, int rng, int fn, int m, bool res, bool cl) {
  if (dtype == 0) return rng == 0 ? swarm_kernel_f64_ref(fn, m, res, cl) : swarm_kernel_f64_philox(fn, m, res, cl);
  return rng == 0 ? swarm_kernel_f32_ref(fn, m, res, cl) : swarm_kernel_f32_philox(fn, m, res, cl);
}

const void* seq_kernel_f64_ref(int fn, int m, bool res);
const void* seq_kernel_f64_philox(int fn, int m, bool res);
const void* seq_kernel_f32_ref(int fn, int m, bool res);
const void* seq_kernel_f32_philox(int fn, int m, bool res);

inline const void* seq_kernel(int dtype, int rng, int fn, int m, bool res) {
  if (dtype == 0) return rng == 0 ? seq_kernel_f64_ref(fn, m, res) : seq_kernel_f64_philox(fn, m, res);
  return rng == 0 ? seq_kernel_f32_ref(fn, m, res) : seq_kernel_f32_philox(fn, m, res);
}

inline const void* chain_kernel(int dtype, int rng, int fn, int m, bool init, bool full) {
  if (dtype == 0)
    return rng == 0 ? chain_kernel_f64_ref(fn, m, init, full) : chain_kernel_f64_philox(fn, m, init, full);
  return rng == 0 ? chain_kernel_f32_ref(fn, m, init, full) : chain_kernel_f32_philox(fn, m, init, full);
}

inline const void* tile_kernel(int dtype, int rng, int fn, int vec, bool fused) {
  if (dtype == 0)
    return rng == 0 ? tile_kernel_f64_ref(fn, vec, fused) : tile_kernel_f64_philox(fn, vec, fused);
  return rng == 0 ? tile_kernel_f32_ref(fn, vec, fused) : tile_kernel_f32_philox(fn, vec, fused);
}
}  // namespace psso
