// inst_e64.cu — step-loop kernels for 64^3 tiles (inst.cuh).
#include "inst.cuh"

PLBM_INSTANTIATE(64)
