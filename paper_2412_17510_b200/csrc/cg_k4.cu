// Device CG for K = 4.
#include "cg1r_inst.cuh"
MPSG_INSTANTIATE_CG(4)
