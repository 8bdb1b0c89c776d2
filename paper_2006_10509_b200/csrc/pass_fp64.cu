#define CGH_T double
#include "dispatch_impl.cuh"
