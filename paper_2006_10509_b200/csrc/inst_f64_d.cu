// Kernel instantiations: double lines of 1024 points.
#include "dispatch_n.cuh"
namespace cgh {
CGH_INSTANTIATE(double, 1024)
}
