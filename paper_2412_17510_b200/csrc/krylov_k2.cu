// Device solve() (all Krylov methods) for K = 2.
#include "krylov_inst.cuh"
MPSG_INSTANTIATE_KRYLOV(2)
