// Microbenchmark (calibration, not product code): legacy warp-level tensor-core MMA
// (mma.sync.m16n8k16 bf16 -> fp32, SASS HMMA) throughput per SM on this GPU, W warps per SM,
// 8 independent accumulator chains per warp.  Reports FLOP/clk/SM and TFLOP/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void mma_kernel(float *out, int iters, long long *cyc) {
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    float c[8][4] = {};
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    long long t1 = clock64();
    float s = 0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out; long long *cyc; cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8);
    for (int w : {4, 8, 12, 16}) {
        const int iters = 4000;
        mma_kernel<<<sms, 32 * w>>>(out, iters, cyc);
        cudaDeviceSynchronize();
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        mma_kernel<<<sms, 32 * w>>>(out, iters, cyc);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const double flop_sm = (double)w * iters * 8 * 16 * 8 * 16 * 2;
        printf("warps/SM=%2d  %.0f FLOP/clk/SM  %.1f TFLOP/s (chip)\n", w, flop_sm / c, flop_sm * sms / (ms * 1e-3) / 1e12);
    }
    return 0;
}
