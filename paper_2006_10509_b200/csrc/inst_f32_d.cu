// Kernel instantiations: float lines of 1024 points.
#include "dispatch_n.cuh"
namespace cgh {
CGH_INSTANTIATE(float, 1024)
}
