// k_swarm instantiations: T=float, RNG=Philox4x32-10.
#define PSSO_T float
#define PSSO_RNG 1
#define PSSO_NAME(x) x##_f32_philox
#include "psso_swarm_inst.cuh"
