// Explicit instantiations of the pair-sweep kernel (d = 3, fused = true), one
// translation unit per slice so the library builds in parallel.  See ca_kernels.cuh.
#include "ca_sweep.cuh"

#define X(D, NM, F) template cudaError_t ca::sweep_launch<D, NM, F>(const ca::Dev&, unsigned, cudaStream_t);
X(3, 9, true) X(3, 11, true) X(3, 13, true)
