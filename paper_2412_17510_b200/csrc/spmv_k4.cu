// SpMV kernels and launcher for K = 4.
#include "spmv_inst.cuh"
MPSG_INSTANTIATE_SPMV(4)
