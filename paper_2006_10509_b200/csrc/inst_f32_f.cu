// Kernel instantiations: float lines of 4096 points.
#include "dispatch_n.cuh"
namespace cgh {
CGH_INSTANTIATE(float, 4096)
}
