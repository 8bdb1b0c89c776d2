// Kernel instantiations: float lines of 512 points.
#include "dispatch_n.cuh"
namespace cgh {
CGH_INSTANTIATE(float, 512)
}
