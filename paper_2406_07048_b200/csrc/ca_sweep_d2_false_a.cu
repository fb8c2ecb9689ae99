// Explicit instantiations of the pair-sweep kernel (d = 2, fused = false), one
// translation unit per slice so the library builds in parallel.  See ca_kernels.cuh.
#include "ca_sweep.cuh"

#define X(D, NM, F) template cudaError_t ca::sweep_launch<D, NM, F>(const ca::Dev&, unsigned, cudaStream_t);
X(2, 9, false) X(2, 11, false) X(2, 13, false)
