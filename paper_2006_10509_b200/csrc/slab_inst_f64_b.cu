// Slab line-pass instantiations: double, N = 2048, 4096.
#include "slab_kernels.cuh"
CGH_SLAB_INSTANTIATE(double, 2048)
CGH_SLAB_INSTANTIATE(double, 4096)
