// Kernel instantiations: float lines of 2048 points.
#include "dispatch_n.cuh"
namespace cgh {
CGH_INSTANTIATE(float, 2048)
}
