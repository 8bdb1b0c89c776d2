// Slab line-pass instantiations: float, N = 16384.
#include "slab_kernels.cuh"
CGH_SLAB_INSTANTIATE(float, 16384)
