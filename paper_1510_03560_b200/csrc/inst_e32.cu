// inst_e32.cu — step-loop kernels for 32^3 tiles (inst.cuh).
#include "inst.cuh"

PLBM_INSTANTIATE(32)
