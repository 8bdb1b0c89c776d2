// Slab line-pass instantiations: float, N = 64, 128, 256, 512, 1024.
#include "slab_kernels.cuh"
CGH_SLAB_INSTANTIATE(float, 64)
CGH_SLAB_INSTANTIATE(float, 128)
CGH_SLAB_INSTANTIATE(float, 256)
CGH_SLAB_INSTANTIATE(float, 512)
CGH_SLAB_INSTANTIATE(float, 1024)
