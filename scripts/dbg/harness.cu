// standalone probe of f3d::k_smooth2 / k_restrict on a small 3D field (variants via -D)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "kf3d.cuh"
int main(int argc, char **argv) {
    int n = argc > 1 ? atoi(argv[1]) : 31, pitch = n + 1, zc = argc > 2 ? atoi(argv[2]) : n;
    size_t el = (size_t)n * n * pitch;
    double *u, *b, *o;
    cudaMalloc(&u, el * 8); cudaMalloc(&b, el * 8); cudaMalloc(&o, el * 8);
    std::vector<double> h(el);
    for (size_t i = 0; i < el; ++i) h[i] = (double)(i % 97) * 0.01;
    cudaMemcpy(u, h.data(), el * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(b, h.data(), el * 8, cudaMemcpyHostToDevice);
    CUtensorMap mu, mb;
    tma_make_map(&mu, u, n, pitch, n, f3d::S_UW, f3d::S_UH, 1);
    tma_make_map(&mb, b, n, pitch, n, f3d::S_BW, f3d::S_BH, 1);
    cudaError_t e0 = cudaFuncSetAttribute(f3d::k_smooth2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f3d::S_SMEM);
    SCoef c{1.0, 0.1, 0.01, 0.5};
    int tx = (n + f3d::S_TX - 1) / f3d::S_TX;
    dim3 grd(tx, tx, (n + zc - 1) / zc);
    f3d::k_smooth2<<<grd, f3d::NT, f3d::S_SMEM>>>(mu, mb, o, n, pitch, (long long)n * pitch, c, zc);
    cudaError_t e1 = cudaGetLastError();
    cudaError_t e2 = cudaDeviceSynchronize();
    printf("%s n=%d zc=%d smem=%zu attr=%s launch=%s sync=%s\n", argv[0], n, zc, f3d::S_SMEM, cudaGetErrorString(e0),
           cudaGetErrorString(e1), cudaGetErrorString(e2));
    return 0;
}
