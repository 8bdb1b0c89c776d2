// Kernel instantiations: float lines of 2, 4, 8, 16, 32, 64 points.
#include "dispatch_n.cuh"
namespace cgh {
CGH_INSTANTIATE(float, 2)
CGH_INSTANTIATE(float, 4)
CGH_INSTANTIATE(float, 8)
CGH_INSTANTIATE(float, 16)
CGH_INSTANTIATE(float, 32)
CGH_INSTANTIATE(float, 64)
}
