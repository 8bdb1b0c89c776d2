// Kernel instantiations: double lines of 128, 256 points.
#include "dispatch_n.cuh"
namespace cgh {
CGH_INSTANTIATE(double, 128)
CGH_INSTANTIATE(double, 256)
}
