// microbenchmark: does SHFL consume L1 data-pipe (shared) wavefronts? compare with LDS.
#include <cstdio>
__global__ void k_shfl(double* out, int iters) {
    double a = threadIdx.x * 1.0, acc = 0.0;
    for (int i = 0; i < iters; ++i) {
        acc += __shfl_sync(0xffffffffu, a, (threadIdx.x + i) & 31);
        a = acc * 0.5;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_lds(double* out, int iters) {
    __shared__ double s[1024];
    s[threadIdx.x] = threadIdx.x;
    __syncthreads();
    double acc = 0.0;
    for (int i = 0; i < iters; ++i) {
        acc += s[(threadIdx.x + i) & 1023];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    double* d;
    cudaMalloc(&d, 148 * 8 * 1024 * 8);
    k_shfl<<<148 * 8, 1024>>>(d, 1000);
    k_lds<<<148 * 8, 1024>>>(d, 1000);
    cudaDeviceSynchronize();
    printf("ok\n");
}
