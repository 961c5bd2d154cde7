// kernels_fast.cuh -- tuned fine-level kernels (placeholder: generic kernels until the tiled
// versions land).
#pragma once
#include "kernels_generic.cuh"

inline void fast_jacobi2d(double *out, const double *in, const double *b, const GridDesc &g, const SCoef &c,
                          cudaStream_t s) {
    dim3 blk(32, 8, 1), grd((g.n + 31) / 32, (g.n + 7) / 8, 1);
    k_jacobi<2><<<grd, blk, 0, s>>>(out, in, b, g, c);
}
inline void fast_jacobi3d(double *out, const double *in, const double *b, const GridDesc &g, const SCoef &c,
                          cudaStream_t s) {
    dim3 blk(32, 8, 1), grd((g.n + 31) / 32, (g.n + 7) / 8, g.n);
    k_jacobi<3><<<grd, blk, 0, s>>>(out, in, b, g, c);
}
