// Slab line-pass instantiations: float, N = 2048, 4096.
#include "slab_kernels.cuh"
CGH_SLAB_INSTANTIATE(float, 2048)
CGH_SLAB_INSTANTIATE(float, 4096)
