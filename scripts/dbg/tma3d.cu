// standalone probe: 3D TMA box loads at various (possibly out-of-range) coordinates
#include <cstdio>
#include <cstdlib>
#include "../../paper_1401_7824_b200/csrc/tma.cuh"
__global__ void k(const __grid_constant__ CUtensorMap m, double *out, int x, int y, int z, int bytes) {
    __shared__ __align__(128) double buf[34 * 34];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    __syncthreads();
    if (threadIdx.x == 0) { mbar_expect_tx(&bar, bytes); tma_load_3d(buf, &m, x, y, z, &bar); }
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < 34 * 34; i += blockDim.x) out[i] = buf[i];
}
int main(int argc, char **argv) {
    int n = 31, pitch = 32, bx = atoi(argv[1]), by = atoi(argv[2]);
    int x = atoi(argv[3]), y = atoi(argv[4]), z = atoi(argv[5]);
    double *f, *o;
    cudaMalloc(&f, (size_t)n * n * pitch * 8);
    cudaMalloc(&o, 34 * 34 * 8);
    cudaMemset(f, 0, (size_t)n * n * pitch * 8);
    CUtensorMap m;
    bool ok = tma_make_map(&m, f, n, pitch, n, bx, by, 1);
    k<<<1, 128>>>(m, o, x, y, z, bx * by * 8);
    cudaError_t e = cudaDeviceSynchronize();
    printf("box %dx%d at (%d,%d,%d): map %d -> %s\n", bx, by, x, y, z, ok, cudaGetErrorString(e));
    return 0;
}
