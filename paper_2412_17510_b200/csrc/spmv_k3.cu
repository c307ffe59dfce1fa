// SpMV kernels and launcher for K = 3.
#include "spmv_inst.cuh"
MPSG_INSTANTIATE_SPMV(3)
