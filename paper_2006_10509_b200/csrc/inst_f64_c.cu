// Kernel instantiations: double lines of 512 points.
#include "dispatch_n.cuh"
namespace cgh {
CGH_INSTANTIATE(double, 512)
}
