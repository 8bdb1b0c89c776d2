#define CGH_T float
#include "dispatch_impl.cuh"
