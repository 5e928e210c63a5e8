// inst_e16.cu — step-loop kernels for 16^3 tiles (inst.cuh).
#include "inst.cuh"

PLBM_INSTANTIATE(16)
