// Device solve() (all Krylov methods) for K = 4.
#include "krylov_inst.cuh"
MPSG_INSTANTIATE_KRYLOV(4)
