// Device CG for K = 2.
#include "cg_inst.cuh"
MPSG_INSTANTIATE_CG(2)
