// psso_tiles_inst.cuh -- kernel instantiation table for one (T, RNG) pair.
// Included by psso_tiles_{f64,f32}_{ref,philox}.cu with PSSO_T, PSSO_RNG,
// PSSO_VEC (16-byte vector width) and PSSO_NAME(x) defined; the four
// translation units compile in parallel.
#include "psso_device.cuh"
#include "psso_registry.h"

namespace psso {

#define PSSO_TILE(FN)                                                                       \
  case FN:                                                                                  \
    if (fused)                                                                              \
      return vec == PSSO_VEC ? (const void*)k_fused<PSSO_T, FN, PSSO_RNG, PSSO_VEC>        \
                             : (const void*)k_tile<PSSO_T, FN, PSSO_RNG, 1, true>;         \
    return vec == PSSO_VEC ? (const void*)k_tile<PSSO_T, FN, PSSO_RNG, PSSO_VEC, false>    \
                           : (const void*)k_tile<PSSO_T, FN, PSSO_RNG, 1, false>;

const void* PSSO_NAME(tile_kernel)(int fn, int vec, bool fused) {
  switch (fn) {
    PSSO_TILE(0) PSSO_TILE(1) PSSO_TILE(2) PSSO_TILE(3) PSSO_TILE(4)
    PSSO_TILE(5) PSSO_TILE(6) PSSO_TILE(7) PSSO_TILE(8) PSSO_TILE(9)
    default:
      return nullptr;
  }
}

// k_chain<.., M, INIT, FULL>: FULL (D == 8*M) only for the iteration kernel
#define PSSO_CHAIN_M(FN, M)                                                                 \
  if (m == M) {                                                                             \
    if (init) return (const void*)k_chain<PSSO_T, FN, PSSO_RNG, M, true, false>;           \
    return full ? (const void*)k_chain<PSSO_T, FN, PSSO_RNG, M, false, true>               \
                : (const void*)k_chain<PSSO_T, FN, PSSO_RNG, M, false, false>;             \
  }
#define PSSO_CHAIN(FN) \
  case FN:             \
    PSSO_CHAIN_M(FN, 4) PSSO_CHAIN_M(FN, 8) PSSO_CHAIN_M(FN, 16) return nullptr;

const void* PSSO_NAME(chain_kernel)(int fn, int m, bool init, bool full) {
  switch (fn) {
    PSSO_CHAIN(0) PSSO_CHAIN(1) PSSO_CHAIN(2) PSSO_CHAIN(3) PSSO_CHAIN(4) PSSO_CHAIN(5)
    PSSO_CHAIN(6) PSSO_CHAIN(7) PSSO_CHAIN(8) PSSO_CHAIN(9)
    default:
      return nullptr;
  }
}

#define PSSO_ROWS(FN)                                                 \
  case FN:                                                            \
    if (w == 1) return (const void*)k_rows<PSSO_T, FN, PSSO_RNG, 1>;  \
    if (w == 2) return (const void*)k_rows<PSSO_T, FN, PSSO_RNG, 2>;  \
    if (w == 4) return (const void*)k_rows<PSSO_T, FN, PSSO_RNG, 4>;  \
    if (w == 8) return (const void*)k_rows<PSSO_T, FN, PSSO_RNG, 8>;  \
    return nullptr;

const void* PSSO_NAME(rows_kernel)(int fn, int w) {
  switch (fn) {
    PSSO_ROWS(0) PSSO_ROWS(1) PSSO_ROWS(2) PSSO_ROWS(5) PSSO_ROWS(6) PSSO_ROWS(9)
    default:
      return nullptr;
  }
}

}  // namespace psso
