// k_tile instantiations: T=float, RNG=philox (all objectives, vector and scalar rows).
#include "psso_device.cuh"
#include "psso_registry.h"

namespace psso {

#define PSSO_TILE(FN)                                                          \
  case FN:                                                                     \
    if (fused)                                                                 \
      return vec == 4 ? (const void*)k_fused<float, FN, 1, 4>                \
                      : (const void*)k_tile<float, FN, 1, 1, true>;                 \
    return vec == 4 ? (const void*)k_tile<float, FN, 1, 4, false>                 \
                    : (const void*)k_tile<float, FN, 1, 1, false>;

const void* tile_kernel_f32_philox(int fn, int vec, bool fused) {
  switch (fn) {
    PSSO_TILE(0) PSSO_TILE(1) PSSO_TILE(2) PSSO_TILE(3) PSSO_TILE(4)
    PSSO_TILE(5) PSSO_TILE(6) PSSO_TILE(7) PSSO_TILE(8) PSSO_TILE(9)
    default:
      return nullptr;
  }
}

#define PSSO_CHAIN(FN)                                                             \
  case FN:                                                                         \
    if (m == 4) return init ? (const void*)k_chain<float, FN, 1, 4, true>           \
                            : (const void*)k_chain<float, FN, 1, 4, false>;          \
    if (m == 8) return init ? (const void*)k_chain<float, FN, 1, 8, true>           \
                            : (const void*)k_chain<float, FN, 1, 8, false>;          \
    if (m == 16) return init ? (const void*)k_chain<float, FN, 1, 16, true>         \
                             : (const void*)k_chain<float, FN, 1, 16, false>;        \
    return nullptr;

const void* chain_kernel_f32_philox(int fn, int m, bool init) {
  switch (fn) {
    PSSO_CHAIN(0) PSSO_CHAIN(1) PSSO_CHAIN(2) PSSO_CHAIN(4) PSSO_CHAIN(5) PSSO_CHAIN(6)
    PSSO_CHAIN(9)
    default:
      return nullptr;
  }
}

}  // namespace psso
