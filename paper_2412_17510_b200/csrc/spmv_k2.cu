// SpMV kernels and launcher for K = 2.
#include "spmv_inst.cuh"
MPSG_INSTANTIATE_SPMV(2)
