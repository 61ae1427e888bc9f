// Microbenchmark: tcgen05.mma issue-to-completion rate on every SM (one CTA per SM), for the
// shapes K1 uses.  SS = both operands from shared memory, TS = A from TMEM (K1's P.V).
// Optional competing shared-memory traffic from other warps (ld.shared.v4 loop), to see how
// much of the tensor pipe's smem operand bandwidth the softmax / converter warps can steal.
// Prints cycles per MMA instruction and dense FLOP/clk/SM.  (Calibration for DESIGN.md.)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2509_02121_b200/csrc tools/umma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.h"
using namespace halo;

constexpr int SMEM = 200 * 1024;

// mode: 0 SS N=64, 1 SS N=128, 2 SS N=256, 3 TS N=128 (K=16 f16), 4 TS N=64, 5 SS N=128 with
// A = 2 alternating 128-row tiles (K1's two sub-tiles sharing K)
__global__ void __launch_bounds__(256, 1) k(int mode, int iters, int noise, long long *cyc, float *sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < SMEM / 16; i += blockDim.x) reinterpret_cast<uint4 *>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
    if (warp == 0) ptx::tmem_alloc(&tslot, 512);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    volatile int *stop = reinterpret_cast<volatile int *>(sm + SMEM - 16);
    if (threadIdx.x == 0) {
        const uint32_t base = ptx::smem_u32(sm);
        const int N = mode == 0 || mode == 4 ? 64 : mode == 2 ? 256 : 128;
        const uint32_t idS = ptx::idesc_bf16(128, N, false, false);
        const uint32_t idT = ptx::idesc_f16(128, N, 0u, 0u, false, true);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
                if (mode <= 2 || mode == 5) {
                    const uint32_t a = base + (mode == 5 ? (it & 1) * 32768 : 0) + off;
                    ptx::mma_bf16_ss(tmem + (mode == 5 ? (it & 1) * 128 : 0), ptx::smem_desc_sw128(a, 16, 1024),
                                     ptx::smem_desc_sw128(base + 65536 + off, 16, 1024), idS, kk > 0);
                } else {
                    ptx::mma_f16_ts(tmem + 256, tmem + kk * 8, ptx::smem_desc_sw128(base + 65536 + kk * 2048, 16384, 1024),
                                    idT, kk > 0);
                }
            }
        }
        ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) *cyc = t1 - t0;
        *stop = 1;
    } else if (noise && warp >= 1) {
        // competing smem reads (16 B per lane per instruction) over the upper 64 KB
        uint4 acc = make_uint4(0, 0, 0, 0);
        const uint4 *p = reinterpret_cast<const uint4 *>(sm + 131072);
        int i = threadIdx.x;
        while (!*stop) {
#pragma unroll 8
            for (int j = 0; j < 64; ++j) {
                uint4 v = p[(i + j * 256) & 4095];
                acc.x ^= v.x; acc.y += v.y;
            }
            i += 7;
        }
        sink[blockIdx.x * blockDim.x + threadIdx.x] = (float)(acc.x + acc.y);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long *cyc; float *sink;
    cudaMalloc(&cyc, 8); cudaMalloc(&sink, 1 << 22);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    const char *names[] = {"SS M128 N64  K16 bf16", "SS M128 N128 K16 bf16", "SS M128 N256 K16 bf16",
                           "TS M128 N128 K16 f16 ", "TS M128 N64  K16 f16 ", "SS M128 N128 2 A tiles"};
    const int Ns[] = {64, 128, 256, 128, 64, 128};
    for (int noise = 0; noise < 2; ++noise)
        for (int mode = 0; mode < 6; ++mode) {
            const int iters = 2000;
            k<<<sms, 256, SMEM>>>(mode, 50, noise, cyc, sink);
            k<<<sms, 256, SMEM>>>(mode, iters, noise, cyc, sink);
            long long c = 0;
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            const double per = (double)c / (iters * 8.0);
            const double flop = 2.0 * 128 * Ns[mode] * 16;
            printf("%s noise=%d: %7.1f cyc/MMA  %7.0f FLOP/clk/SM  (floor %d cyc)  %s\n", names[mode], noise, per,
                   flop / per, 128 * Ns[mode] / 256, cudaGetErrorString(e));
        }
    return 0;
}
