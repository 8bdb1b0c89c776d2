// Kernel instantiations: double lines of 2, 4, 8, 16, 32, 64 points.
#include "dispatch_n.cuh"
namespace cgh {
CGH_INSTANTIATE(double, 2)
CGH_INSTANTIATE(double, 4)
CGH_INSTANTIATE(double, 8)
CGH_INSTANTIATE(double, 16)
CGH_INSTANTIATE(double, 32)
CGH_INSTANTIATE(double, 64)
}
