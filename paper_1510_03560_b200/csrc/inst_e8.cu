// inst_e8.cu — step-loop kernels for 8^3 tiles (inst.cuh).
#include "inst.cuh"

PLBM_INSTANTIATE(8)
