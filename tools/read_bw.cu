// Read-bandwidth microbenchmark (calibration for DESIGN.md; not product code):
//  (a) contiguous stream of N bytes with LDG.128, grid = k x SMs
//  (b) 4-KiB slabs at 32-KiB stride (the K2 pattern: one kv head of consecutive blocks)
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
__global__ void rd_contig(const int4 *__restrict__ p, long long n16, int *out) {
    int acc = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x) {
        int4 v = __ldg(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678) out[0] = acc;
}
// each warp reads slabs of 4 KiB: slab s at byte offset (s / 8) * 32K + (s % 8) * 4K ... ordered
// so that a warp walks one head's slabs (stride 32 KiB)
__global__ void rd_slabs(const int4 *__restrict__ p, long long nslabs, int *out) {
    int acc = 0;
    const int lane = threadIdx.x & 31;
    long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long s = w; s < nslabs; s += nw) {
        long long head = s % 8, blk = s / 8;   // walk: consecutive warps take consecutive heads
        const int4 *slab = p + (blk * 8 + head) * 256;  // 4 KiB = 256 x int4
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            int4 v = __ldg(slab + i * 32 + lane);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    if (acc == 0x12345678) out[0] = acc;
}
// K2-shaped streaming: per warp a ring of STAGES x 8 KiB (K slab + V slab), lane 0 issues
// two 4-KiB cp.async.bulk per stage, all lanes wait on the stage mbarrier and XOR the data.
template <int WARPS, int STAGES>
__global__ void __launch_bounds__(WARPS * 32, 1) rd_bulk(const uint8_t *__restrict__ k, const uint8_t *__restrict__ v,
                                                        long long nslabs, int *out) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t *ring = sm + warp * (STAGES * 8192 + 64);
    unsigned long long *bar = (unsigned long long *)(ring + STAGES * 8192);
    if (lane == 0) for (int s = 0; s < STAGES; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(bar + s)));
    __syncwarp();
    long long gw = blockIdx.x * (long long)WARPS + warp, nw = (long long)gridDim.x * WARPS;
    long long per = (nslabs + nw - 1) / nw, s0 = gw * per, s1 = s0 + per < nslabs ? s0 + per : nslabs;
    int acc = 0;
    long long issued = s0, done = s0;
    auto issue = [&](long long s) {
        int st = (int)((s - s0) % STAGES);
        unsigned dst = (unsigned)__cvta_generic_to_shared(ring + st * 8192);
        unsigned b = (unsigned)__cvta_generic_to_shared(bar + st);
        long long head = s % 8, blk = s / 8;
        const uint8_t *gk = k + (blk * 8 + head) * 4096, *gv = v + (blk * 8 + head) * 4096;
        if (lane == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 8192;" ::"r"(b));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(dst), "l"(gk), "r"(b));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(dst + 4096), "l"(gv), "r"(b));
        }
    };
    for (; issued < s1 && issued < s0 + STAGES; ++issued) issue(issued);
    for (; done < s1; ++done) {
        int st = (int)((done - s0) % STAGES);
        unsigned par = (unsigned)(((done - s0) / STAGES) & 1);
        unsigned b = (unsigned)__cvta_generic_to_shared(bar + st);
        unsigned ok = 0;
        while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(b), "r"(par));
        const int4 *d = (const int4 *)(ring + st * 8192);
#pragma unroll
        for (int i = 0; i < 16; ++i) { int4 x = d[i * 32 + lane]; acc ^= x.x ^ x.y ^ x.z ^ x.w; }
        __syncwarp();
        if (issued < s1) { issue(issued); ++issued; }
    }
    if (acc == 0x12345678) out[0] = acc;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t bytes = (size_t)4 << 30;
    int4 *p; int *o; cudaMalloc(&p, bytes); cudaMalloc(&o, 4); cudaMemset(p, 1, bytes);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int k : {2, 4, 8, 16}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a); rd_contig<<<sms * k, 256>>>(p, bytes / 16, o); cudaEventRecord(b);
            cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("contig  grid=%3dxSM  %.0f GB/s\n", k, bytes / ms / 1e6);
        }
    }
    for (int k : {2, 4, 8, 16}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a); rd_slabs<<<sms * k, 256>>>(p, bytes / 4096, o); cudaEventRecord(b);
            cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("slabs   grid=%3dxSM  %.0f GB/s\n", k, bytes / ms / 1e6);
        }
    }
    // 283 MB (the K2 C1 footprint) cold: flush L2 with a 512 MB memset in between
    const size_t small = 283ull << 20;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(p + bytes / 32, rep, bytes / 2);
        cudaEventRecord(a); rd_slabs<<<sms * 8, 256>>>(p, small / 4096, o); cudaEventRecord(b);
        cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
        printf("slabs 283MB cold  %.1f us  %.0f GB/s\n", ms * 1e3, small / ms / 1e6);
    }
    // K2-shaped bulk streaming over 283 MB (K half + V half), back to back
    {
        const size_t per2 = 283ull << 20;
        const long long nsl = per2 / 8192;  // (K slab, V slab) pairs
        auto run = [&](auto kern, int warps, int stages, const char *name) {
            int smem = warps * (stages * 8192 + 64);
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            float best = 1e9;
            for (int i = 0; i < 6; ++i) {
                const uint8_t *base = (const uint8_t *)p + (size_t)(i % 6) * per2;
                cudaEventRecord(a); kern<<<sms, warps * 32, smem>>>(base, base + per2 / 2, nsl, o); cudaEventRecord(b);
                cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (i) best = ms < best ? ms : best;
            }
            printf("bulk %-14s %.1f us  %.0f GB/s\n", name, best * 1e3, per2 / best / 1e6);
        };
        run(rd_bulk<12, 2>, 12, 2, "12w x 2st");
        run(rd_bulk<8, 3>, 8, 3, "8w x 3st");
        run(rd_bulk<6, 4>, 6, 4, "6w x 4st");
        run(rd_bulk<4, 6>, 4, 6, "4w x 6st");
        run(rd_bulk<16, 1>, 16, 1, "16w x 1st");
    }
    // layer-by-layer: 12 distinct 283 MB buffers read back to back (no dirty L2 lines)
    const size_t per = 283ull << 20;
    const int nbuf = (int)(bytes / per);
    cudaEvent_t ev[16];
    for (int i = 0; i <= nbuf; ++i) cudaEventCreate(&ev[i]);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(ev[0]);
        for (int i = 0; i < nbuf; ++i) {
            rd_slabs<<<sms * 8, 256>>>(p + i * (per / 16), per / 4096, o);
            cudaEventRecord(ev[i + 1]);
        }
        cudaEventSynchronize(ev[nbuf]);
        float tot; cudaEventElapsedTime(&tot, ev[0], ev[nbuf]);
        printf("back-to-back %d x 283MB: %.1f us each, %.0f GB/s;", nbuf, tot * 1e3 / nbuf, nbuf * per / tot / 1e6);
        for (int i = 1; i < 4; ++i) { float m; cudaEventElapsedTime(&m, ev[i], ev[i+1]); printf(" %.1f", m * 1e3); }
        printf("\n");
    }
    return 0;
}
