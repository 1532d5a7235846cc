// k_swarm instantiations: T=double, RNG=reference (keyed SplitMix64).
#define PSSO_T double
#define PSSO_RNG 0
#define PSSO_NAME(x) x##_f64_ref
#include "psso_swarm_inst.cuh"
