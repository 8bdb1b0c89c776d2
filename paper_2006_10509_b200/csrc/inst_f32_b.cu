// Kernel instantiations: float lines of 128, 256 points.
#include "dispatch_n.cuh"
namespace cgh {
CGH_INSTANTIATE(float, 128)
CGH_INSTANTIATE(float, 256)
}
