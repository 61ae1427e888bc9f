// Microbenchmark: warp-instruction throughput of MUFU.EX2, F2FP (f32x2->f16x2), FFMA2, FFMA
// on one B200 SM-full launch.  Prints ops/clk/SM.  (Calibration for DESIGN.md; not product.)
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(float *out, int iters, long long *cyc) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
    unsigned u[8] = {0};
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
            if (OP == 1) { asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(a[i]), "f"(a[(i + 1) & 7]));
                           a[i] = __uint_as_float(u[i] ^ 0x3f800000u); }
            if (OP == 2) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
            if (OP == 3) { unsigned long long x = *(unsigned long long*)&a[i & 6];
                asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(x)); *(unsigned long long*)&a[i & 6] = x; }
            if (OP == 4) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
                           asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(a[i]), "f"(a[(i + 1) & 7]));
                           a[(i+4)&7] = __uint_as_float(u[i] ^ 0x3f800000u); }
            if (OP == 5) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(a[(i+3)&7]));
            if (OP == 6) { unsigned short lo = (unsigned short)(u[i] + i), hi = (unsigned short)(u[i] >> 3);
                asm volatile("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(a[i]) : "h"(lo), "h"(hi)); }
            if (OP == 7) { unsigned w = __float_as_uint(a[(i + 5) & 7]);
                a[i] += __uint_as_float(w << 16) + __uint_as_float(w & 0xFFFF0000u); }
        }
    }
    long long t1 = clock64();
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + u[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out; long long *cyc; cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8);
    const char *names[] = {"MUFU.EX2 f32", "F2FP f16x2", "FFMA", "FFMA2 (2 flops-pairs)", "MUFU.EX2+F2FP f16 pair", "FMNMX", "FHFMA.BF16 (mixed f32<-bf16*bf16)", "bf16x2->2xf32 cvt + 2 FADD"};
    for (int op = 0; op < 8; ++op) {
        for (int warps : {4, 8, 16}) {
            int iters = 4096;
            auto launch = [&]() {
                if (op == 0) k<0><<<sms, warps * 32>>>(out, iters, cyc);
                if (op == 1) k<1><<<sms, warps * 32>>>(out, iters, cyc);
                if (op == 2) k<2><<<sms, warps * 32>>>(out, iters, cyc);
                if (op == 3) k<3><<<sms, warps * 32>>>(out, iters, cyc);
                if (op == 4) k<4><<<sms, warps * 32>>>(out, iters, cyc);
                if (op == 5) k<5><<<sms, warps * 32>>>(out, iters, cyc);
                if (op == 6) k<6><<<sms, warps * 32>>>(out, iters, cyc);
                if (op == 7) k<7><<<sms, warps * 32>>>(out, iters, cyc);
            };
            launch(); cudaDeviceSynchronize();
            launch(); cudaDeviceSynchronize();
            long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            double ops = (double)iters * 8 * warps * 32;  // per SM (one CTA per SM)
            printf("%-22s warps/SM=%2d  %.2f thread-ops/clk/SM\n", names[op], warps, ops / c);
        }
    }
    return 0;
}
