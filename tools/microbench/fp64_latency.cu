// microbenchmark: dependent-chain latency and single-warp / full-SM throughput of fp64 ops on this
// GPU (DFMA, DMUL, DADD, MUFU.RSQ64H), clock64 cycles per operation.
#include <cstdio>
#include <cstdint>

template <int OP>
__global__ void chain(double* out, long long* cyc, int iters, double seed) {
    double a = seed + threadIdx.x * 1e-3, b = 1.0000001, c = 1e-9;
    __syncwarp();
    const long long t0 = clock64();
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (OP == 0) a = fma(a, b, c);
            else if (OP == 1) a = a * b;
            else if (OP == 2) a = a + c;
            else { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a)); a = r + 1.0; }
        }
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
__global__ void indep(double* out, long long* cyc, int iters, double seed) {  // 8 independent chains
    double a[8];
    for (int j = 0; j < 8; ++j) a[j] = seed + threadIdx.x * 1e-3 + j;
    const double b = 1.0000001, c = 1e-9;
    const long long t0 = clock64();
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (OP == 0) a[j] = fma(a[j], b, c);
                else if (OP == 1) a[j] = a[j] * b;
                else a[j] = a[j] + c;
            }
    }
    const long long t1 = clock64();
    double s = 0;
    for (int j = 0; j < 8; ++j) s += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    double* out; long long* cyc; cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 1 << 16);
    const int iters = 4096;
    const char* names[4] = {"DFMA", "DMUL", "DADD", "MUFU.RSQ64H+DADD"};
    for (int op = 0; op < 4; ++op) {
        long long h;
        for (int rep = 0; rep < 2; ++rep) {
            if (op == 0) chain<0><<<1, 32>>>(out, cyc, iters, 1.0);
            if (op == 1) chain<1><<<1, 32>>>(out, cyc, iters, 1.0);
            if (op == 2) chain<2><<<1, 32>>>(out, cyc, iters, 1.0);
            if (op == 3) chain<3><<<1, 32>>>(out, cyc, iters, 1.0);
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        }
        printf("%-18s dependent latency: %.2f cycles/op (1 warp)\n", names[op], double(h) / (iters * 16));
    }
    for (int op = 0; op < 3; ++op) {
        for (int w : {1, 4, 16}) {
            long long h;
            for (int rep = 0; rep < 2; ++rep) {
                if (op == 0) indep<0><<<1, 32 * w>>>(out, cyc, iters, 1.0);
                if (op == 1) indep<1><<<1, 32 * w>>>(out, cyc, iters, 1.0);
                if (op == 2) indep<2><<<1, 32 * w>>>(out, cyc, iters, 1.0);
                cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            }
            const double ops = double(iters) * 16 * w;  // warp instructions issued by the SM
            printf("%-5s %2d warps x 8 chains: %.2f cycles per warp instruction per SM\n", names[op], w, double(h) / ops);
        }
    }
    return 0;
}
