// Kernel instantiations: double lines of 4096 points.
#include "dispatch_n.cuh"
namespace cgh {
CGH_INSTANTIATE(double, 4096)
}
