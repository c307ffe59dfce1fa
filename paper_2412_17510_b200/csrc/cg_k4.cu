// Device CG for K = 4.
#include "cg_inst.cuh"
MPSG_INSTANTIATE_CG(4)
