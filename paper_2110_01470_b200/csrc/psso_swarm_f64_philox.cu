// k_swarm instantiations: T=double, RNG=Philox4x32-10.
#define PSSO_T double
#define PSSO_RNG 1
#define PSSO_NAME(x) x##_f64_philox
#include "psso_swarm_inst.cuh"
