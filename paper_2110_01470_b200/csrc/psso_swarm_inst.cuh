// psso_swarm_inst.cuh -- k_swarm instantiations for one (T, RNG) pair.
// Included by psso_swarm_{f64,f32}_{ref,philox}.cu with PSSO_T, PSSO_RNG and
// PSSO_NAME(x) defined.
#include "psso_seq.cuh"
#include "psso_swarm.cuh"
#include "psso_registry.h"

namespace psso {

#define PSSO_SWARM_M(FN, M)                                                                    \
  if (m == M) {                                                                                \
    if (cl) return res ? (const void*)k_swarm<PSSO_T, FN, PSSO_RNG, M, true, true> : nullptr;  \
    return res ? (const void*)k_swarm<PSSO_T, FN, PSSO_RNG, M, true, false>                    \
               : (const void*)k_swarm<PSSO_T, FN, PSSO_RNG, M, false, false>;                  \
  }
#define PSSO_SWARM(FN) \
  case FN:             \
    PSSO_SWARM_M(FN, 4) PSSO_SWARM_M(FN, 8) PSSO_SWARM_M(FN, 16) return nullptr;

const void* PSSO_NAME(swarm_kernel)(int fn, int m, bool res, bool cl) {
  switch (fn) {
    PSSO_SWARM(0) PSSO_SWARM(1) PSSO_SWARM(2) PSSO_SWARM(3) PSSO_SWARM(4)
    PSSO_SWARM(5) PSSO_SWARM(6) PSSO_SWARM(7) PSSO_SWARM(8) PSSO_SWARM(9)
    default:
      return nullptr;
  }
}

#define PSSO_SEQ_M(FN, M)                                                          \
  if (m == M) return res ? (const void*)k_seq<PSSO_T, FN, PSSO_RNG, M, true>        \
                         : (const void*)k_seq<PSSO_T, FN, PSSO_RNG, M, false>;
#define PSSO_SEQ(FN) \
  case FN:           \
    PSSO_SEQ_M(FN, 4) PSSO_SEQ_M(FN, 8) PSSO_SEQ_M(FN, 16) return nullptr;

const void* PSSO_NAME(seq_kernel)(int fn, int m, bool res) {
  switch (fn) {
    PSSO_SEQ(0) PSSO_SEQ(1) PSSO_SEQ(2) PSSO_SEQ(3) PSSO_SEQ(4)
    PSSO_SEQ(5) PSSO_SEQ(6) PSSO_SEQ(7) PSSO_SEQ(8) PSSO_SEQ(9)
    default:
      return nullptr;
  }
}

}  // namespace psso
