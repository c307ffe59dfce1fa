// Device CG for K = 3.
#include "cg1r_inst.cuh"
MPSG_INSTANTIATE_CG(3)
