// general.cu -- generally-K-sparse solver kernels (collision vote, pruning,
// subspace pursuit).  Filled in by the general-path milestone.
#include "common.cuh"
#include "general.cuh"
