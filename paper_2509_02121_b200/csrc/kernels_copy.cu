// K4 (pack / unpack) and K5 (append) -- bitwise KV copies between the exchange layout
// [layer][token][kv_head][d] (standardised KV state at operator boundaries)
// and the paged pool [layer][block][kv_head][16][d] (block-level management).
//
// HBM-bound: every byte is read once and written once with 16-byte vector accesses.
// Thread layout: one CTA row covers `tpb` tokens x (hkv heads x d/8 chunks); a thread's
// (head, chunk, token lane) is fixed, so the only per-iteration index math is one slot
// load and two multiply-adds.  Consecutive lanes touch consecutive 16-B chunks of a
// token row, so both sides are coalesced (256-B runs per head at d=128).  Each thread
// keeps kUnroll independent loads in flight; gridDim.x x layers is sized to a multiple
// of the SM count.
#include "halo_internal.h"

#include <algorithm>

namespace halo {
namespace {

constexpr int kUnroll = 4;

__device__ __forceinline__ int4 ld_stream(const int4 *p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// bf16 bits of max |x| over the 8 bf16 of a 16-B chunk (magnitude bits order like the values).
__device__ __forceinline__ uint32_t absmax8(int4 w) {
    const uint32_t a = max(max((uint32_t)w.x & 0x7fffu, ((uint32_t)w.x >> 16) & 0x7fffu),
                           max((uint32_t)w.y & 0x7fffu, ((uint32_t)w.y >> 16) & 0x7fffu));
    const uint32_t b = max(max((uint32_t)w.z & 0x7fffu, ((uint32_t)w.z >> 16) & 0x7fffu),
                           max((uint32_t)w.w & 0x7fffu, ((uint32_t)w.w >> 16) & 0x7fffu));
    return max(a, b);
}

// Block-wide max of m (256 threads), valid in thread 0.
__device__ __forceinline__ uint32_t cta_max256(uint32_t m) {
    __shared__ uint32_t red[8];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0)
        for (int i = 1; i < 8; ++i) m = max(m, red[i]);
    __syncthreads();
    return m;
}

struct Geo {
    int64_t n;          // tokens addressed
    int32_t hkv, cpr;   // heads, 16-B chunks per head row (d/8)
    int32_t tpb;        // tokens per CTA iteration
    int64_t pool_layer; // int4 chunks per pool layer
    int64_t src_rows;   // rows per layer in the exchange tensor
};

// Pool chunk of (layer, slot, head h, chunk e): ((layer*cap + blk)*hkv + h)*16 + off rows.
__device__ __forceinline__ int64_t pool_chunk(const Geo &g, int layer, int32_t slot, int h,
                                              int e) {
    const int64_t blk = slot >> 4, off = slot & 15;
    return (int64_t)layer * g.pool_layer + ((blk * g.hkv + h) * 16 + off) * g.cpr + e;
}

// src/dst exchange rows: [layer][i][h][chunk]
__global__ void kv_scatter_kernel(int4 *__restrict__ pk, int4 *__restrict__ pv,
                                  const int4 *__restrict__ sk, const int4 *__restrict__ sv,
                                  Geo g, const int32_t *__restrict__ slots,
                                  const uint32_t *__restrict__ tags, uint64_t *__restrict__ vmax,
                                  int64_t cap, int64_t n_copy, int layer_begin) {
    const int inner = g.hkv * g.cpr;
    const int lane_tok = threadIdx.x / inner;
    if (lane_tok >= g.tpb) return;
    const int h = (threadIdx.x % inner) / g.cpr, e = threadIdx.x % g.cpr;
    const int layer = layer_begin + blockIdx.y;
    const int64_t step = (int64_t)gridDim.x * g.tpb;
    const int64_t src_layer = (int64_t)blockIdx.y * g.src_rows;
    for (int64_t i0 = (int64_t)blockIdx.x * g.tpb + lane_tok; i0 < g.n; i0 += step * kUnroll) {
        int4 vk[kUnroll], vv[kUnroll];
        int64_t dst[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int64_t i = i0 + u * step;
            dst[u] = -1;
            if (i < g.n) {
                dst[u] = pool_chunk(g, layer, slots[i], h, e);
                if (i < n_copy) {
                    const int64_t s = ((src_layer + i) * g.hkv + h) * g.cpr + e;
                    vk[u] = ld_stream(sk + s);
                    vv[u] = ld_stream(sv + s);
                } else {
                    vk[u] = make_int4(0, 0, 0, 0);
                    vv[u] = vk[u];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (dst[u] >= 0) {
                pk[dst[u]] = vk[u];
                pv[dst[u]] = vv[u];
            }
        }
        if (tags) {  // V-table: max |V| per (layer, block), lanes of one block reduced first
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const int64_t i = i0 + u * step;
                const int32_t blk = i < g.n ? (slots[i] >> 4) : -1;
                const uint32_t m = blk >= 0 ? absmax8(vv[u]) : 0u;
                const uint32_t act = __activemask();
                if (inner % 32 == 0 && act == 0xffffffffu) {
                    // a whole warp lies in one token row (one block): one reduction, one atomic
                    const uint32_t red = __reduce_max_sync(act, m);
                    if (blk >= 0 && (threadIdx.x & 31) == 0)
                        atomicMax(reinterpret_cast<unsigned long long *>(vmax + (int64_t)layer * cap + blk),
                                  (unsigned long long)vmax_entry(tags[i], red));
                    continue;
                }
                const uint32_t grp = __match_any_sync(act, blk);
                const uint32_t red = __reduce_max_sync(grp, m);
                if (blk >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1)
                    atomicMax(reinterpret_cast<unsigned long long *>(vmax + (int64_t)layer * cap + blk),
                              (unsigned long long)vmax_entry(tags[i], red));
            }
        }
    }
}

__global__ void kv_gather_kernel(const int4 *__restrict__ pk, const int4 *__restrict__ pv,
                                 int4 *__restrict__ dk, int4 *__restrict__ dv, Geo g,
                                 const int32_t *__restrict__ slots, int layer_begin) {
    const int inner = g.hkv * g.cpr;
    const int lane_tok = threadIdx.x / inner;
    if (lane_tok >= g.tpb) return;
    const int h = (threadIdx.x % inner) / g.cpr, e = threadIdx.x % g.cpr;
    const int layer = layer_begin + blockIdx.y;
    const int64_t step = (int64_t)gridDim.x * g.tpb;
    const int64_t dst_layer = (int64_t)blockIdx.y * g.n;
    for (int64_t i0 = (int64_t)blockIdx.x * g.tpb + lane_tok; i0 < g.n; i0 += step * kUnroll) {
        int4 vk[kUnroll], vv[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int64_t i = i0 + u * step;
            if (i < g.n) {
                const int64_t s = pool_chunk(g, layer, slots[i], h, e);
                vk[u] = ld_stream(pk + s);
                vv[u] = ld_stream(pv + s);
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int64_t i = i0 + u * step;
            if (i < g.n) {
                const int64_t d = ((dst_layer + i) * g.hkv + h) * g.cpr + e;
                dk[d] = vk[u];
                dv[d] = vv[u];
            }
        }
    }
}

// Block shape: `inner` = hkv*cpr threads per token; up to 256 threads (or one token row
// if wider).  Grid: enough CTAs per layer that layers x gx ~ 8 CTAs per SM.
void shape(const PoolGeom &pg, int64_t n, int layers, int num_sms, Geo &g, dim3 &grid,
           int &threads) {
    g.hkv = pg.hkv;
    g.cpr = pg.d / 8;
    const int inner = g.hkv * g.cpr;
    g.tpb = inner >= 256 ? 1 : 256 / inner;
    threads = g.tpb * inner;
    g.n = n;
    g.pool_layer = pg.cap * pg.hkv * 16 * g.cpr;
    const int64_t per_layer_ctas = (n + (int64_t)g.tpb * kUnroll - 1) / ((int64_t)g.tpb * kUnroll);
    int64_t want = ((int64_t)num_sms * 8 + layers - 1) / layers;
    if (want > per_layer_ctas) want = per_layer_ctas;
    if (want < 1) want = 1;
    grid = dim3((unsigned)want, (unsigned)layers, 1);
}

// Pool-to-pool block copy (same device): pair i copies pool block src_blk[i] of every
// layer in [layer_begin, layer_end) to block dst_blk[i] of the destination pool, K and V.
// A (layer, block) of all heads is one contiguous run of hkv*16*d*2 bytes on both sides
// (32 KiB at hkv=8, d=128), so this is a plain streaming copy: 16-B loads, kCopyUnroll in
// flight per thread, the grid a multiple of the SM count.
constexpr int kCopyUnroll = 8;
__global__ void __launch_bounds__(256) kv_copy_blocks_kernel(
    const int4 *__restrict__ sk, const int4 *__restrict__ sv, int4 *__restrict__ dk,
    int4 *__restrict__ dv, const int32_t *__restrict__ pairs, const uint32_t *__restrict__ dst_tags,
    const uint64_t *__restrict__ src_vmax, uint64_t *__restrict__ dst_vmax, int64_t src_cap,
    int64_t dst_cap, int64_t nitems, int32_t nblk, int32_t run16, int64_t src_layer16,
    int64_t dst_layer16, int layer_begin) {
    // item = ((layer - layer_begin) * nblk + pair) * 2 + (K|V): one contiguous run of run16 int4
    for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
        const int kv = (int)(item & 1);
        const int64_t lp = item >> 1;
        const int32_t pr = (int32_t)(lp % nblk);
        const int64_t layer = layer_begin + lp / nblk;
        const int4 *src = (kv ? sv : sk) + layer * src_layer16 + (int64_t)pairs[2 * pr] * run16;
        int4 *dst = (kv ? dv : dk) + layer * dst_layer16 + (int64_t)pairs[2 * pr + 1] * run16;
        if (kv && threadIdx.x == 0)
            dst_vmax[layer * dst_cap + pairs[2 * pr + 1]] =
                vmax_entry(dst_tags[pr], (uint32_t)src_vmax[layer * src_cap + pairs[2 * pr]]);
        for (int o0 = threadIdx.x; o0 < run16; o0 += 256 * kCopyUnroll) {
            int4 v[kCopyUnroll];
#pragma unroll
            for (int u = 0; u < kCopyUnroll; ++u)
                if (o0 + u * 256 < run16) v[u] = ld_stream(src + o0 + u * 256);
#pragma unroll
            for (int u = 0; u < kCopyUnroll; ++u)
                if (o0 + u * 256 < run16) dst[o0 + u * 256] = v[u];
        }
    }
}

// K4 pack / unpack for migration, block-granular: item j of [item_begin, item_end) is the
// (layer j / nblk, node block blocks[j % nblk]) pair; its K run and its V run (hkv*16*d*2
// bytes each, contiguous in the pool) go to / come from the wire buffer at
// ((j - item_begin) * 2 + kv) * run16 int4.  A whole block moves, the zero tail of a partial
// last block included, so the destination slab is bit-identical to the source slab.
__global__ void __launch_bounds__(256) kv_runs_kernel(
    int4 *__restrict__ pk, int4 *__restrict__ pv, int4 *__restrict__ buf,
    const int32_t *__restrict__ blocks, const uint32_t *__restrict__ tags, uint64_t *__restrict__ vmax,
    int64_t cap, int32_t nblk, int64_t item_begin, int64_t nitems2, int32_t run16,
    int64_t pool_layer16, int to_pool) {
    for (int64_t it = blockIdx.x; it < nitems2; it += gridDim.x) {
        const int kv = (int)(it & 1);
        const int64_t j = item_begin + (it >> 1);
        const int64_t layer = j / nblk;
        int4 *pool = (kv ? pv : pk) + layer * pool_layer16 + (int64_t)blocks[j % nblk] * run16;
        int4 *wire = buf + it * run16;
        const int4 *src = to_pool ? wire : pool;
        int4 *dst = to_pool ? pool : wire;
        uint32_t m = 0;
        for (int o0 = threadIdx.x; o0 < run16; o0 += 256 * kCopyUnroll) {
            int4 v[kCopyUnroll];
#pragma unroll
            for (int u = 0; u < kCopyUnroll; ++u)
                if (o0 + u * 256 < run16) v[u] = ld_stream(src + o0 + u * 256);
#pragma unroll
            for (int u = 0; u < kCopyUnroll; ++u)
                if (o0 + u * 256 < run16) {
                    dst[o0 + u * 256] = v[u];
                    m = max(m, absmax8(v[u]));
                }
        }
        if (to_pool && kv) {  // the block's V-table entry (a whole block arrived)
            m = cta_max256(m);
            if (threadIdx.x == 0) vmax[layer * cap + blocks[j % nblk]] = vmax_entry(tags[j % nblk], m);
        }
    }
}

// V-table entries recomputed from the pool: one CTA per (layer, block).
__global__ void __launch_bounds__(256) kv_vmax_kernel(const int4 *__restrict__ pv, const int32_t *__restrict__ blocks,
                                                      const uint32_t *__restrict__ tags, uint64_t *__restrict__ vmax,
                                                      int64_t cap, int32_t nblk, int64_t nitems, int32_t run16) {
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        const int64_t layer = it / nblk;
        const int32_t b = blocks[it % nblk];
        const int4 *src = pv + (layer * cap + b) * run16;
        uint32_t m = 0;
        for (int o = threadIdx.x; o < run16; o += 256) m = max(m, absmax8(ld_stream(src + o)));
        m = cta_max256(m);
        if (threadIdx.x == 0) vmax[layer * cap + b] = vmax_entry(tags[it % nblk], m);
    }
}

}  // namespace

cudaError_t launch_kv_copy_blocks(const PoolGeom &sg, const void *src_k, const void *src_v,
                                  const PoolGeom &dg, void *dst_k, void *dst_v,
                                  const int32_t *pairs, const uint32_t *dst_tags, int32_t nblk,
                                  int layer_begin, int layer_end, int num_sms, cudaStream_t s) {
    const int layers = layer_end - layer_begin;
    if (nblk == 0 || layers <= 0) return cudaSuccess;
    const int32_t run16 = sg.hkv * kBlockTok * sg.d * 2 / 16;  // int4 chunks per (layer, block)
    const int64_t nitems = (int64_t)layers * nblk * 2;
    int64_t grid = nitems;
    const int64_t cap = (int64_t)num_sms * 8;  // 8 CTAs of 256 threads per SM
    if (grid > cap) grid = cap;
    kv_copy_blocks_kernel<<<(unsigned)grid, 256, 0, s>>>(
        (const int4 *)src_k, (const int4 *)src_v, (int4 *)dst_k, (int4 *)dst_v, pairs, dst_tags,
        sg.vmax, dg.vmax, sg.cap, dg.cap, nitems, nblk, run16, sg.cap * run16, dg.cap * run16,
        layer_begin);
    return cudaGetLastError();
}

cudaError_t launch_kv_scatter(const PoolGeom &pg, void *pool_k, void *pool_v, const void *src_k,
                              const void *src_v, int64_t src_rows, const int32_t *slots,
                              const uint32_t *tags, int64_t n_copy, int64_t n_zero, int layer_begin,
                              int layer_end, int num_sms, cudaStream_t s) {
    const int64_t n = n_copy + n_zero;
    const int layers = layer_end - layer_begin;
    if (n == 0 || layers <= 0) return cudaSuccess;
    Geo g;
    dim3 grid;
    int threads;
    shape(pg, n, layers, num_sms, g, grid, threads);
    g.src_rows = src_rows;
    kv_scatter_kernel<<<grid, threads, 0, s>>>((int4 *)pool_k, (int4 *)pool_v,
                                               (const int4 *)src_k, (const int4 *)src_v, g,
                                               slots, tags, pg.vmax, pg.cap, n_copy, layer_begin);
    return cudaGetLastError();
}

cudaError_t launch_kv_gather(const PoolGeom &pg, const void *pool_k, const void *pool_v,
                             void *dst_k, void *dst_v, const int32_t *slots, int64_t n,
                             int layer_begin, int layer_end, int num_sms, cudaStream_t s) {
    const int layers = layer_end - layer_begin;
    if (n == 0 || layers <= 0) return cudaSuccess;
    Geo g;
    dim3 grid;
    int threads;
    shape(pg, n, layers, num_sms, g, grid, threads);
    g.src_rows = n;
    kv_gather_kernel<<<grid, threads, 0, s>>>((const int4 *)pool_k, (const int4 *)pool_v,
                                              (int4 *)dst_k, (int4 *)dst_v, g, slots,
                                              layer_begin);
    return cudaGetLastError();
}

cudaError_t launch_kv_runs(const PoolGeom &pg, void *pool_k, void *pool_v, void *buf,
                           const int32_t *blocks, const uint32_t *tags, int32_t nblk,
                           int64_t item_begin, int64_t item_end, bool to_pool, int max_ctas,
                           cudaStream_t s) {
    const int64_t nitems2 = 2 * (item_end - item_begin);
    if (nblk == 0 || nitems2 <= 0) return cudaSuccess;
    const int32_t run16 = pg.hkv * kBlockTok * pg.d * 2 / 16;
    int64_t grid = nitems2;
    if (grid > max_ctas) grid = max_ctas;
    kv_runs_kernel<<<(unsigned)grid, 256, 0, s>>>((int4 *)pool_k, (int4 *)pool_v, (int4 *)buf, blocks, tags,
                                                  pg.vmax, pg.cap, nblk, item_begin, nitems2, run16,
                                                  pg.cap * run16, to_pool ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_kv_vmax(const PoolGeom &pg, const void *pool_v, const int32_t *blocks,
                           const uint32_t *tags, int32_t nblk, int num_sms, cudaStream_t s) {
    const int64_t nitems = (int64_t)pg.layers * nblk;
    if (nitems == 0) return cudaSuccess;
    const int32_t run16 = pg.hkv * kBlockTok * pg.d * 2 / 16;
    int64_t grid = std::min<int64_t>(nitems, (int64_t)num_sms * 8);
    kv_vmax_kernel<<<(unsigned)grid, 256, 0, s>>>((const int4 *)pool_v, blocks, tags, pg.vmax, pg.cap, nblk,
                                                  nitems, run16);
    return cudaGetLastError();
}

namespace {
// Host -> device copy by the SMs from mapped pinned memory (zero-copy reads over PCIe): the
// small per-step uploads (plan arrays, slot lists) then never queue behind a large transfer
// on a copy engine (e.g. a background prefetch of a prefix node).
__global__ void __launch_bounds__(256) h2d_small_kernel(const int4 *__restrict__ src, int4 *__restrict__ dst, int64_t n16,
                                                        const uint8_t *__restrict__ srcb, uint8_t *__restrict__ dstb,
                                                        int64_t tail_off, int tail) {
    for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n16; i += (int64_t)gridDim.x * 256) dst[i] = src[i];
    if (blockIdx.x == 0 && threadIdx.x < tail) dstb[tail_off + threadIdx.x] = srcb[tail_off + threadIdx.x];
}
}  // namespace

cudaError_t launch_h2d_small(const void *mapped_src, void *dst, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return cudaSuccess;
    const int64_t n16 = (int64_t)(bytes / 16);
    const int tail = (int)(bytes % 16);
    int64_t grid = (n16 + 255) / 256;
    if (grid > 64) grid = 64;
    if (grid < 1) grid = 1;
    h2d_small_kernel<<<(unsigned)grid, 256, 0, s>>>((const int4 *)mapped_src, (int4 *)dst, n16,
                                                    (const uint8_t *)mapped_src, (uint8_t *)dst, n16 * 16, tail);
    return cudaGetLastError();
}

}  // namespace halo
