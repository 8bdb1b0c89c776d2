// Slab line-pass instantiations: float, N = 8192.
#include "slab_kernels.cuh"
CGH_SLAB_INSTANTIATE(float, 8192)
