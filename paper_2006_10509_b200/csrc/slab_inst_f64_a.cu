// Slab line-pass instantiations: double, N = 64, 128, 256, 512, 1024.
#include "slab_kernels.cuh"
CGH_SLAB_INSTANTIATE(double, 64)
CGH_SLAB_INSTANTIATE(double, 128)
CGH_SLAB_INSTANTIATE(double, 256)
CGH_SLAB_INSTANTIATE(double, 512)
CGH_SLAB_INSTANTIATE(double, 1024)
