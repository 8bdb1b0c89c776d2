// Slab line-pass instantiations: double, N = 8192.
#include "slab_kernels.cuh"
CGH_SLAB_INSTANTIATE(double, 8192)
