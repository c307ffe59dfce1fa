// Device CG for K = 2.
#include "cg1r_inst.cuh"
MPSG_INSTANTIATE_CG(2)
