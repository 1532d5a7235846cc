// k_tile instantiations: T=float, RNG=ref (all objectives, vector and scalar rows).
#include "psso_device.cuh"
#include "psso_registry.h"

namespace psso {

#define PSSO_TILE(FN)                                              \
  case FN:                                                         \
    return vec == 4 ? (const void*)k_tile<float, FN, 0, 4>          \
                     : (const void*)k_tile<float, FN, 0, 1>;

const void* tile_kernel_f32_ref(int fn, int vec) {
  switch (fn) {
    PSSO_TILE(0) PSSO_TILE(1) PSSO_TILE(2) PSSO_TILE(3) PSSO_TILE(4)
    PSSO_TILE(5) PSSO_TILE(6) PSSO_TILE(7) PSSO_TILE(8) PSSO_TILE(9)
    default:
      return nullptr;
  }
}

}  // namespace psso
