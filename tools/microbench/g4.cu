// microbenchmark: TMA tile::gather4 of 32-B rows (SWIZZLE_32B) vs direct 256-bit LDG gathers.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <bool MATH>
__global__ void __launch_bounds__(32) k_direct(const double4* __restrict__ a, const double4* __restrict__ b,
                                                const double4* __restrict__ c, const uint32_t* idx, int nchunks, double* out) {
    double acc = 0.0;
    const int lane = threadIdx.x;
    for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const uint32_t j = idx[ch * 32 + lane];
        double4 x, y, z;
        asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(x.x), "=d"(x.y), "=d"(x.z), "=d"(x.w) : "l"(a + j));
        asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(y.x), "=d"(y.y), "=d"(y.z), "=d"(y.w) : "l"(b + j));
        asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(z.x), "=d"(z.y), "=d"(z.z), "=d"(z.w) : "l"(c + j));
        double s = x.x + x.y + x.z + x.w + y.x + y.y + y.z + y.w + z.x + z.y + z.z + z.w;
        if (MATH) for (int it = 0; it < 40; ++it) s = s * 0.999999 + 1e-9;
        acc += s;
    }
    out[blockIdx.x * 32 + lane] = acc;
}

struct __align__(256) Buf {
    double4 r[3][32];
};

__global__ void __launch_bounds__(32) k_tma(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                                             const __grid_constant__ CUtensorMap tc, const uint32_t* idx, int nchunks,
                                             double* out) {
    __shared__ Buf buf;
    __shared__ __align__(8) uint64_t bar;
    const int lane = threadIdx.x;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    double acc = 0.0;
    uint32_t phase = 0;
    for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const uint32_t j = idx[ch * 32 + lane];
        // lanes 0..23: array lane/8, rows of contact lanes 4(lane%8) .. +3
        const int arr = lane >> 3, g = lane & 7;
        const uint32_t r0 = __shfl_sync(0xffffffffu, j, 4 * g), r1 = __shfl_sync(0xffffffffu, j, 4 * g + 1);
        const uint32_t r2 = __shfl_sync(0xffffffffu, j, 4 * g + 2), r3 = __shfl_sync(0xffffffffu, j, 4 * g + 3);
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(3 * 32 * 32));
        __syncwarp();
        if (lane < 24) {
            const CUtensorMap* tm = arr == 0 ? &ta : (arr == 1 ? &tb : &tc);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                ::"r"(smem_u32(&buf.r[arr][4 * g])), "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(&bar)),
                  "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
                : "memory");
        }
        // wait for the phase
        uint32_t done = 0;
        while (!done) {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(smem_u32(&bar)), "r"(phase) : "memory");
        }
        phase ^= 1u;
        // read own rows (SWIZZLE_32B: 16-B chunk bit 4 ^= address bit 7)
        double s = 0.0;
        for (int k = 0; k < 3; ++k) {
            const char* base = reinterpret_cast<const char*>(&buf.r[k][0]);
            for (int h = 0; h < 2; ++h) {
                const uint32_t off = 32u * lane + 16u * h;
                const uint32_t sw = off ^ (((off >> 7) & 1u) << 4);
                const double2 v = *reinterpret_cast<const double2*>(base + sw);
                s += v.x + v.y;
            }
        }
        acc += s;
        __syncwarp();
    }
    out[blockIdx.x * 32 + lane] = acc;
}


__global__ void __launch_bounds__(32) k_tma2(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                                              const __grid_constant__ CUtensorMap tc, const uint32_t* idx, int nchunks,
                                              double* out) {
    __shared__ Buf buf[2];
    __shared__ __align__(8) uint64_t bar[2];
    const int lane = threadIdx.x;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    const int arr = lane >> 3, g = lane & 7;
    auto issue = [&](int ch, int sb) {
        const uint32_t j = idx[ch * 32 + lane];
        const uint32_t r0 = __shfl_sync(0xffffffffu, j, 4 * g), r1 = __shfl_sync(0xffffffffu, j, 4 * g + 1);
        const uint32_t r2 = __shfl_sync(0xffffffffu, j, 4 * g + 2), r3 = __shfl_sync(0xffffffffu, j, 4 * g + 3);
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[sb])), "r"(3 * 32 * 32));
        __syncwarp();
        if (lane < 24) {
            const CUtensorMap* tm = arr == 0 ? &ta : (arr == 1 ? &tb : &tc);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                ::"r"(smem_u32(&buf[sb].r[arr][4 * g])), "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(&bar[sb])),
                  "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
                : "memory");
        }
    };
    double acc = 0.0;
    uint32_t ph[2] = {0, 0};
    int sb = 0;
    int ch = blockIdx.x;
    if (ch < nchunks) issue(ch, 0);
    for (; ch < nchunks; ch += gridDim.x) {
        if (ch + (int)gridDim.x < nchunks) issue(ch + gridDim.x, sb ^ 1);
        uint32_t done = 0;
        while (!done) {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(smem_u32(&bar[sb])), "r"(ph[sb]) : "memory");
        }
        ph[sb] ^= 1u;
        double s = 0.0;
        for (int k = 0; k < 3; ++k) {
            const char* base = reinterpret_cast<const char*>(&buf[sb].r[k][0]);
            for (int h = 0; h < 2; ++h) {
                const uint32_t off = 32u * lane + 16u * h;
                const uint32_t sw = off ^ (((off >> 7) & 1u) << 4);
                const double2 v = *reinterpret_cast<const double2*>(base + sw);
                s += v.x + v.y;
            }
        }
        // some math to overlap (~ the force kernel has thousands of cycles per chunk)
        for (int it = 0; it < 40; ++it) s = s * 0.999999 + 1e-9;
        acc += s;
        __syncwarp();
        sb ^= 1;
    }
    out[blockIdx.x * 32 + lane] = acc;
}


// AoS 112-B records (14 doubles): one gather4 per 4 contacts, 8 per chunk
struct __align__(1024) BufA { double r[32][16]; };
__global__ void __launch_bounds__(32) k_tma_aos(const __grid_constant__ CUtensorMap tr, const uint32_t* idx, int nchunks,
                                                 double* out) {
    __shared__ BufA buf[2];
    __shared__ __align__(8) uint64_t bar[2];
    const int lane = threadIdx.x;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    const int g = lane & 7;
    auto issue = [&](int ch, int sb) {
        const uint32_t j = idx[ch * 32 + lane];
        const uint32_t r0 = __shfl_sync(0xffffffffu, j, 4 * g), r1 = __shfl_sync(0xffffffffu, j, 4 * g + 1);
        const uint32_t r2 = __shfl_sync(0xffffffffu, j, 4 * g + 2), r3 = __shfl_sync(0xffffffffu, j, 4 * g + 3);
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[sb])), "r"(32 * 128));
        __syncwarp();
        if (lane < 8) {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                ::"r"(smem_u32(&buf[sb].r[4 * g][0])), "l"(reinterpret_cast<uint64_t>(&tr)), "r"(smem_u32(&bar[sb])),
                  "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
                : "memory");
        }
    };
    double acc = 0.0;
    uint32_t ph[2] = {0, 0};
    int sb = 0;
    int ch = blockIdx.x;
    if (ch < nchunks) issue(ch, 0);
    for (; ch < nchunks; ch += gridDim.x) {
        if (ch + (int)gridDim.x < nchunks) issue(ch + gridDim.x, sb ^ 1);
        uint32_t done = 0;
        while (!done) {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(smem_u32(&bar[sb])), "r"(ph[sb]) : "memory");
        }
        ph[sb] ^= 1u;
        double s = 0.0;
        const double2* row = reinterpret_cast<const double2*>(&buf[sb].r[lane][0]);
        for (int h = 0; h < 6; ++h) { const double2 v = row[h ^ (lane & 7)]; s += v.x + v.y; }
        for (int it = 0; it < 40; ++it) s = s * 0.999999 + 1e-9;
        acc += s;
        __syncwarp();
        sb ^= 1;
    }
    out[blockIdx.x * 32 + lane] = acc;
}

int main() {
    const int N = 1 << 20, nch = 1 << 17;
    std::vector<double4> h(N);
    for (int i = 0; i < N; ++i) h[i] = make_double4(i, i * 2.0, i * 3.0, i * 4.0);
    std::vector<uint32_t> hi(nch * 32);
    uint64_t st = 88172645463325252ull;
    for (size_t k = 0; k < hi.size(); ++k) {
        st ^= st << 13; st ^= st >> 7; st ^= st << 17;
        const uint32_t base = (k / 32) * 8 % N;  // local neighbourhoods
        hi[k] = (base + static_cast<uint32_t>(st % 8192)) % N;
    }
    double4 *a, *b, *c; uint32_t* idx; double* out;
    cudaMalloc(&a, N * 32); cudaMalloc(&b, N * 32); cudaMalloc(&c, N * 32);
    cudaMalloc(&idx, hi.size() * 4); cudaMalloc(&out, 148 * 16 * 32 * 8 * 2);
    cudaMemcpy(a, h.data(), N * 32, cudaMemcpyHostToDevice);
    cudaMemcpy(b, h.data(), N * 32, cudaMemcpyHostToDevice);
    cudaMemcpy(c, h.data(), N * 32, cudaMemcpyHostToDevice);
    cudaMemcpy(idx, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    CUtensorMap tm[3];
    double4* arrs[3] = {a, b, c};
    for (int k = 0; k < 3; ++k) {
        cuuint64_t dims[2] = {4, (cuuint64_t)N};
        cuuint64_t strides[1] = {32};
        cuuint32_t box[2] = {4, 1};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&tm[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, arrs[k], dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("encode %d -> %d\n", k, (int)r);
    }
    double* aos; cudaMalloc(&aos, (size_t)N * 128);
    {
        std::vector<double> ha((size_t)N * 16);
        for (int i = 0; i < N; ++i) for (int k = 0; k < 12; ++k) ha[(size_t)i * 16 + k] = (&h[i].x)[k % 4];
        cudaMemcpy(aos, ha.data(), (size_t)N * 128, cudaMemcpyHostToDevice);
    }
    CUtensorMap tma_aos;
    {
        cuuint64_t dims[2] = {16, (cuuint64_t)N};
        cuuint64_t strides[1] = {128};
        cuuint32_t box[2] = {16, 1};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&tma_aos, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, aos, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("encode aos -> %d\n", (int)r);
    }
    const int grid = 148 * 16;
    std::vector<double> o1(grid * 32), o2(grid * 32);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        float t1, t2;
        cudaEventRecord(e0); k_direct<false><<<grid, 32>>>(a, b, c, idx, nch, out); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&t1, e0, e1);
        cudaMemcpy(o1.data(), out, grid * 32 * 8, cudaMemcpyDeviceToHost);
        cudaEventRecord(e0); k_tma<<<grid, 32>>>(tm[0], tm[1], tm[2], idx, nch, out); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&t2, e0, e1);
        cudaMemcpy(o2.data(), out, grid * 32 * 8, cudaMemcpyDeviceToHost);
        float t3;
        cudaEventRecord(e0); k_tma2<<<grid, 32>>>(tm[0], tm[1], tm[2], idx, nch, out); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&t3, e0, e1);
        float t4;
        cudaEventRecord(e0); k_direct<true><<<grid, 32>>>(a, b, c, idx, nch, out); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&t4, e0, e1);
        printf("direct +math %.1f us\n", t4 * 1e3);
        float t5;
        cudaEventRecord(e0); k_tma_aos<<<grid, 32>>>(tma_aos, idx, nch, out); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&t5, e0, e1);
        printf("tma aos 128B double-buffered +math %.1f us (%s)\n", t5 * 1e3, cudaGetErrorString(cudaGetLastError()));
        printf("tma double-buffered (+40 dependent DFMA per chunk) %.1f us\n", t3 * 1e3);
        int bad = 0;
        for (int i = 0; i < grid * 32; ++i) bad += o1[i] != o2[i];
        printf("direct %.1f us  tma %.1f us  mismatches %d  err %s\n", t1 * 1e3, t2 * 1e3, bad, cudaGetErrorString(cudaGetLastError()));
    }
}
