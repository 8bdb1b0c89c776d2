// Kernel instantiations: double lines of 2048 points.
#include "dispatch_n.cuh"
namespace cgh {
CGH_INSTANTIATE(double, 2048)
}
