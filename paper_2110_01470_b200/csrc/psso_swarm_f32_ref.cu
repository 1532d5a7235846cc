// k_swarm instantiations: T=float, RNG=reference (keyed SplitMix64).
#define PSSO_T float
#define PSSO_RNG 0
#define PSSO_NAME(x) x##_f32_ref
#include "psso_swarm_inst.cuh"
