// Device solve() (all Krylov methods) for K = 3.
#include "krylov_inst.cuh"
MPSG_INSTANTIATE_KRYLOV(3)
