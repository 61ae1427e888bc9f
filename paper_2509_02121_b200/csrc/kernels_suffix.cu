// K2 + K3: paged-suffix decode attention with the fused log-sum-exp merge.
//
// What it computes (per request r, kv head j, the g q-heads of j): softmax attention of
// the decode query against the request's PRIVATE paged KV (its suffix, plus any prefix
// node the plan folded in because too few requests share it), then the log-sum-exp
// merge with every K1 partial of r's shared prefix path.  The merge makes the result
// identical to unshared attention over the whole context ("Exact answers";
// prefix reuse PAPER.md:343).  Decode is memory-bound (PAPER.md:122 §2.1, :341 §3.3):
// the design goal is HBM bandwidth.
//
// B200 design:
//  * dynamic schedule: the blocks of all (request, kv head) units form one sequence cut
//    into chunks of a few blocks; warps (148 SMs x kK2Warps) take chunks from an atomic
//    queue, so SMs that stream faster take more work and the tail stays short whatever the
//    suffix lengths.  A unit cut by chunk boundaries leaves one partial softmax state per
//    piece; the last piece to finish (atomic arrival counter) merges them in a fixed
//    order -> bit-deterministic results.
//  * warp-level streaming: every warp owns a ring of kStages smem stages; its lane 0 issues
//    one 1-D bulk async copy (cp.async.bulk, TMA engine) per 4-KiB K slab and V slab of a
//    16-token block, completion on a per-stage mbarrier; prefetch runs across unit
//    boundaries.  Each K/V element is read from HBM once for all g q-heads (GQA reuse).
//  * compute from smem on CUDA cores: a token row is split over d/8 lanes (16-B LDS per
//    lane); q.k partial sums of the g heads are combined with a transpose-reduce
//    (log2(d/8)+g-1 shuffles instead of g*log2(d/8)), fp32x2 FMAs (FFMA2) for the dot
//    products and the P.V update, online softmax in base 2 with fp32 state.
//  * K3 epilogue: merge the suffix state with the normalised fp32 K1 partials of the
//    request (slots in a fixed order), write fp32 out and lse.
#include "halo_internal.h"
#include "ptx.h"

#include <cstdlib>

#ifdef HALO_K1_TRACE
// Debug: per-warp [start, first data, end] %globaltimer of the last launch.
__device__ unsigned long long *g_k2_trace = nullptr;
extern "C" int halo_debug_k2_trace(void *buf) {
    return (int)cudaMemcpyToSymbol(g_k2_trace, &buf, sizeof(buf));
}
#define K2_TRACE(slot)                                                                  \
    do {                                                                                \
        if (lane == 0 && g_k2_trace) {                                                  \
            unsigned long long t_;                                                      \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                    \
            g_k2_trace[(blockIdx.x * kWarps + warp) * 4 + (slot)] = t_;                 \
        }                                                                               \
    } while (0)
#else
#define K2_TRACE(slot) do { } while (0)
#endif

namespace halo {
namespace {

constexpr int kWarps = kK2Warps;
constexpr int kStages = 2;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

struct SuffixArgs {
    PlanDev p;
    const uint16_t *pool_k, *pool_v;  // bf16 bits
    int64_t layer_off;                // elements to this layer in the pool
    const uint16_t *q;                // [nreq][hq][D]
    float *out, *lse;
    int32_t hkv, hq;
    float qscale;                     // scale * log2(e)
    int32_t load_mode;                // 0: cp.async.bulk (TMA) per slab, 1: cp.async 16 B per lane
};

template <int D, int G>
struct Shape {
    static constexpr int LPT = D / 8;       // lanes per token row (16-B chunk per lane)
    static constexpr int TPI = 32 / LPT;    // tokens per warp iteration
    static constexpr int NIT = kBlockTok / TPI;
    static constexpr int SLAB = kBlockTok * D * 2;  // bytes of one (block, head) slab
    static constexpr int STAGE = 2 * SLAB;          // K + V
    static constexpr int RING = kStages * STAGE;
    static constexpr int PS = kBlockTok * G * 4;    // p scratch
    static constexpr int CRING = 8;                 // acquired chunk ids (producer -> consumer)
    static constexpr int WARP_SMEM = RING + PS + 16 * 4 + kStages * 8 + CRING * 4;
    static constexpr int WARP_SMEM_AL = (WARP_SMEM + 127) / 128 * 128;
    static_assert(G <= LPT, "transpose-reduce needs g <= d/8");
};

// Sum each of v[0..G) over the LPT lanes of a token group; afterwards lane c holds the
// full sum of head c / (LPT/G) in v[0].
template <int G, int LPT>
__device__ __forceinline__ float transpose_reduce(float (&v)[G], int c) {
    int mask = LPT / 2;
#pragma unroll
    for (int lvl = 0; (G >> lvl) > 1; ++lvl) {
        const int half = (G >> lvl) / 2;
        const bool upper = (c & mask) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
            const float keep = upper ? v[i + half] : v[i];
            const float send = upper ? v[i] : v[i + half];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
        }
        mask >>= 1;
    }
#pragma unroll
    for (int m = LPT / G / 2; m >= 1; m >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], m);
    return v[0];
}

// Final merge of a unit's suffix state (base-2 max mh, sum lh, unnormalised o) with the
// request's K1 partials, then the fp32 output / lse store.  Lanes of token group 0 only.
template <int D, int G>
__device__ __forceinline__ void finalize(const SuffixArgs &a, int req, int head, int c,
                                         const float (&mh)[G], const float (&lh)[G],
                                         float2 (&o2)[G][4]) {
    const PlanDev &P = a.p;
    const int nslots = P.req_nslots[req];
    float M[G], L[G];
#pragma unroll
    for (int h = 0; h < G; ++h) M[h] = (lh[h] > 0.f) ? mh[h] + __log2f(lh[h]) : -INFINITY;
    const int64_t slot_stride = (int64_t)P.nreq * a.hq;
    for (int sl = 0; sl < nslots; ++sl) {
#pragma unroll
        for (int h = 0; h < G; ++h) {
            const float lp = P.part_lse[sl * slot_stride + (int64_t)req * a.hq + head * G + h] * kLog2e;
            M[h] = fmaxf(M[h], lp);
        }
    }
#pragma unroll
    for (int h = 0; h < G; ++h) {
        const float ws = (lh[h] > 0.f) ? ptx::ex2(mh[h] - M[h]) : 0.f;
        L[h] = lh[h] * ws;
#pragma unroll
        for (int i = 0; i < 4; ++i) o2[h][i] = ptx::fmul2(o2[h][i], make_float2(ws, ws));
    }
    for (int sl = 0; sl < nslots; ++sl) {
#pragma unroll
        for (int h = 0; h < G; ++h) {
            const int64_t row = sl * slot_stride + (int64_t)req * a.hq + head * G + h;
            const float w = ptx::ex2(P.part_lse[row] * kLog2e - M[h]);
            L[h] += w;
            const float4 *po = reinterpret_cast<const float4 *>(P.part_o + row * D + c * 8);
            const float4 x0 = po[0], x1 = po[1];
            const float2 ww = make_float2(w, w);
            o2[h][0] = ptx::ffma2(ww, make_float2(x0.x, x0.y), o2[h][0]);
            o2[h][1] = ptx::ffma2(ww, make_float2(x0.z, x0.w), o2[h][1]);
            o2[h][2] = ptx::ffma2(ww, make_float2(x1.x, x1.y), o2[h][2]);
            o2[h][3] = ptx::ffma2(ww, make_float2(x1.z, x1.w), o2[h][3]);
        }
    }
#pragma unroll
    for (int h = 0; h < G; ++h) {
        const float inv = 1.f / L[h];
        float4 *dst = reinterpret_cast<float4 *>(a.out + ((int64_t)req * a.hq + head * G + h) * D + c * 8);
        dst[0] = make_float4(o2[h][0].x * inv, o2[h][0].y * inv, o2[h][1].x * inv, o2[h][1].y * inv);
        dst[1] = make_float4(o2[h][2].x * inv, o2[h][2].y * inv, o2[h][3].x * inv, o2[h][3].y * inv);
        if (a.lse != nullptr && c == h)
            a.lse[(int64_t)req * a.hq + head * G + h] = (M[h] + __log2f(L[h])) * kLn2;
    }
}

template <int D, int G>
__global__ void __launch_bounds__(kWarps * 32, 1) suffix_decode_kernel(const SuffixArgs a) {
    using S = Shape<D, G>;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t *ws = smem_raw + warp * S::WARP_SMEM_AL;
    float *ps = reinterpret_cast<float *>(ws + S::RING);
    float *alph = ps + kBlockTok * G;
    uint64_t *full = reinterpret_cast<uint64_t *>(alph + 16);
    int32_t *cring = reinterpret_cast<int32_t *>(full + kStages);

    K2_TRACE(0);
    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) ptx::mbar_init(&full[s], a.load_mode ? 32 : 1);
        ptx::fence_barrier_init();
    }
    __syncwarp();

    const PlanDev &P = a.p;
    const int hw = lane / S::LPT;   // token group within the warp
    const int c = lane % S::LPT;    // 16-B chunk of the row
    const int hsel = c / (S::LPT / G);
    const bool head_writer = (c % (S::LPT / G)) == 0;
    const int gw = blockIdx.x * kWarps + warp;
    if (gw >= P.nwarps) return;
    const uint16_t *pk = a.pool_k + a.layer_off;
    const uint16_t *pv = a.pool_v + a.layer_off;

    // ---- producer: walks the blocks of the chunks it acquires (all lanes track it) ----
    int pc = -1, phi = 0, px = 0, pu = 0, p_bu = 0, p_eu = 0, p_rb = 0, p_head = 0;
    uint32_t p_count = 0, c_count = 0, p_chunks = 0, c_chunks = 0;
    auto p_load_unit = [&]() {
        p_bu = P.unit_boff[pu];
        p_eu = P.unit_boff[pu + 1];
        const int req = P.unit_req[pu / a.hkv];
        p_head = pu % a.hkv;
        p_rb = P.req_blk_off[req];
    };
    // The first chunk of warp w is chunk w (static: no atomic, neighbouring warps stream
    // neighbouring slabs); later chunks come from the queue, fetched one acquisition ahead
    // so the atomic's latency is hidden.
    // Tail chunks [nwarps, nchunks) are spread over kK2Queues contiguous queues; warp w
    // starts at queue w % kK2Queues and steals from the following queues when it runs dry.
    const int ntail = max(P.nchunks - P.nwarps, 0);
    const int per_q = (ntail + kK2Queues - 1) / kK2Queues;
    int qcur = gw % kK2Queues, qtried = 0;
    auto next_tail = [&]() -> int {
        while (qtried < kK2Queues) {
            const int base = qcur * per_q;
            const int size = min(per_q, ntail - base);
            if (size > 0) {
                const int i = atomicAdd(&P.sched[2 + qcur], 1);
                if (i < size) return P.nwarps + base + i;
            }
            qcur = (qcur + 1) % kK2Queues;
            ++qtried;
        }
        return P.nchunks;
    };
    int next_c = gw;
    auto acquire = [&]() {
        int c = __shfl_sync(0xffffffffu, next_c, 0);
        if (c >= P.nchunks) c = -1;
        else if (lane == 0) next_c = next_tail();
        if (lane == 0) cring[p_chunks % S::CRING] = c;
        ++p_chunks;
        pc = c;
        if (c >= 0) {
            px = P.chunk_lo[c];
            phi = P.chunk_lo[c + 1];
            pu = P.chunk_u0[c];
            p_load_unit();
        }
    };
    acquire();
    auto fill = [&]() {
        while (pc >= 0 && p_count - c_count < (uint32_t)kStages) {
            if (px >= phi) {
                acquire();
                continue;
            }
            while (px >= p_eu) {  // next unit (skips zero-length units)
                ++pu;
                p_load_unit();
            }
            const int st = p_count % kStages;
            uint8_t *dst = ws + st * S::STAGE;
            if (a.load_mode == 0) {
                if (lane == 0) {
                    const uint32_t e = P.req_blk[p_rb + (px - p_bu)];
                    const int64_t off = ((int64_t)(e & kBlkMask) * a.hkv + p_head) * (kBlockTok * D);
                    ptx::mbar_arrive_expect_tx(&full[st], S::STAGE);
                    ptx::bulk_g2s(dst, pk + off, S::SLAB, &full[st]);
                    ptx::bulk_g2s(dst + S::SLAB, pv + off, S::SLAB, &full[st]);
                }
            } else {
                const uint32_t e = P.req_blk[p_rb + (px - p_bu)];
                const int64_t off = ((int64_t)(e & kBlkMask) * a.hkv + p_head) * (kBlockTok * D);
                const uint8_t *gk = reinterpret_cast<const uint8_t *>(pk + off);
                const uint8_t *gv = reinterpret_cast<const uint8_t *>(pv + off);
#pragma unroll
                for (int i = 0; i < S::SLAB / 16 / 32; ++i) {
                    const int o = (i * 32 + lane) * 16;
                    ptx::cp_async16(dst + o, gk + o);
                    ptx::cp_async16(dst + S::SLAB + o, gv + o);
                }
                ptx::cp_async_mbar_arrive(&full[st]);
            }
            ++px;
            ++p_count;
        }
    };
    fill();

    for (;;) {
        fill();  // makes sure the next chunk id has been acquired
        __syncwarp();
        const int cc = cring[c_chunks % S::CRING];
        ++c_chunks;
        if (cc < 0) break;
        const int lo = P.chunk_lo[cc], hi = P.chunk_lo[cc + 1];
        const int u_begin = P.chunk_u0[cc], u_end = P.chunk_u1[cc];
    for (int u = u_begin; u < u_end; ++u) {
        const int bu = P.unit_boff[u], eu = P.unit_boff[u + 1];
        const int xs = max(bu, lo), xe = min(eu, hi);
        const int req = P.unit_req[u / a.hkv];
        const int head = u % a.hkv;
        const int rb = P.req_blk_off[req] - bu;
        // q rows of the g heads of kv head `head`, this lane's 8 dims, pre-scaled.
        float2 q2[G][4];
#pragma unroll
        for (int h = 0; h < G; ++h) {
            const uint4 raw = *reinterpret_cast<const uint4 *>(
                a.q + ((int64_t)req * a.hq + head * G + h) * D + c * 8);
            const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 f = ptx::bf2_to_f2(w[i]);
                q2[h][i] = make_float2(f.x * a.qscale, f.y * a.qscale);
            }
        }
        float m = -INFINITY, l = 0.f;
        float2 o2[G][4];
#pragma unroll
        for (int h = 0; h < G; ++h)
#pragma unroll
            for (int i = 0; i < 4; ++i) o2[h][i] = make_float2(0.f, 0.f);

        for (int x = xs; x < xe; ++x) {
            fill();
            const int st = c_count % kStages;
            const int ntok = (int)(P.req_blk[rb + x] >> kBlkCountShift) + 1;
            ptx::mbar_wait(&full[st], (c_count / kStages) & 1);
            if (c_count == 0) K2_TRACE(1);
            const uint16_t *ks = reinterpret_cast<const uint16_t *>(ws + st * S::STAGE);
            const uint16_t *vs = ks + kBlockTok * D;

            // ---- scores s[it] of head hsel for token it*TPI + hw ----
            float s[S::NIT];
#pragma unroll
            for (int it = 0; it < S::NIT; ++it) {
                const int t = it * S::TPI + hw;
                const uint4 raw = *reinterpret_cast<const uint4 *>(ks + t * D + c * 8);
                const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
                float part[G];
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    float2 acc = ptx::fmul2(q2[h][0], ptx::bf2_to_f2(w[0]));
#pragma unroll
                    for (int i = 1; i < 4; ++i) acc = ptx::ffma2(q2[h][i], ptx::bf2_to_f2(w[i]), acc);
                    part[h] = acc.x + acc.y;
                }
                const float sc = transpose_reduce<G, S::LPT>(part, c);
                s[it] = (t < ntok) ? sc : -INFINITY;
            }
            // ---- online softmax (base 2) for head hsel ----
            float bm = s[0];
#pragma unroll
            for (int it = 1; it < S::NIT; ++it) bm = fmaxf(bm, s[it]);
#pragma unroll
            for (int msk = S::LPT; msk < 32; msk <<= 1)
                bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, msk));
            const float m_new = fmaxf(m, bm);
            const float alpha = ptx::ex2(m - m_new);
            float psum = 0.f;
#pragma unroll
            for (int it = 0; it < S::NIT; ++it) {
                s[it] = ptx::ex2(s[it] - m_new);
                psum += s[it];
            }
#pragma unroll
            for (int msk = S::LPT; msk < 32; msk <<= 1)
                psum += __shfl_xor_sync(0xffffffffu, psum, msk);
            l = l * alpha + psum;
            m = m_new;
            if (head_writer) {
#pragma unroll
                for (int it = 0; it < S::NIT; ++it) ps[(it * S::TPI + hw) * G + hsel] = s[it];
                if (hw == 0) alph[hsel] = alpha;
            }
            __syncwarp();
            // ---- o = o * alpha + P.V ----
#pragma unroll
            for (int h = 0; h < G; ++h) {
                const float al = alph[h];
#pragma unroll
                for (int i = 0; i < 4; ++i) o2[h][i] = ptx::fmul2(o2[h][i], make_float2(al, al));
            }
#pragma unroll
            for (int it = 0; it < S::NIT; ++it) {
                const int t = it * S::TPI + hw;
                if (t < ntok) {
                    const uint4 raw = *reinterpret_cast<const uint4 *>(vs + t * D + c * 8);
                    const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
                    float p[G];
#pragma unroll
                    for (int h = 0; h < G; ++h) p[h] = ps[t * G + h];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float2 v = ptx::bf2_to_f2(w[i]);
#pragma unroll
                        for (int h = 0; h < G; ++h)
                            o2[h][i] = ptx::ffma2(make_float2(p[h], p[h]), v, o2[h][i]);
                    }
                }
            }
            __syncwarp();
            ++c_count;
        }
        fill();

        // ---- combine the TPI token groups ----
#pragma unroll
        for (int msk = S::LPT; msk < 32; msk <<= 1)
#pragma unroll
            for (int h = 0; h < G; ++h)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    o2[h][i].x += __shfl_xor_sync(0xffffffffu, o2[h][i].x, msk);
                    o2[h][i].y += __shfl_xor_sync(0xffffffffu, o2[h][i].y, msk);
                }
        // per-head (m, l) from the lane that owns each head
        float mh[G], lh[G];
#pragma unroll
        for (int h = 0; h < G; ++h) {
            mh[h] = __shfl_sync(0xffffffffu, m, h * (S::LPT / G));
            lh[h] = __shfl_sync(0xffffffffu, l, h * (S::LPT / G));
        }
        const int nseg = P.unit_nseg[u];
        if (nseg == 1) {
            if (hw == 0) finalize<D, G>(a, req, head, c, mh, lh, o2);
        } else {
            // ---- stream-K: publish this piece's state; the last piece merges them all ----
            const int seg = cc - P.unit_chunk0[u];
            const int slot = P.unit_seg[u] + seg;
            if (hw == 0) {
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    float4 *dst = reinterpret_cast<float4 *>(P.seg_o + ((int64_t)slot * G + h) * D + c * 8);
                    dst[0] = make_float4(o2[h][0].x, o2[h][0].y, o2[h][1].x, o2[h][1].y);
                    dst[1] = make_float4(o2[h][2].x, o2[h][2].y, o2[h][3].x, o2[h][3].y);
                }
                if (c < G) *reinterpret_cast<float2 *>(P.seg_ml + ((int64_t)slot * G + c) * 2) = make_float2(mh[c], lh[c]);
            }
            __threadfence();
            __syncwarp();
            int old = 0;
            if (lane == 0) old = atomicAdd(&P.unit_count[u], 1);
            old = __shfl_sync(0xffffffffu, old, 0);
            if (old == nseg - 1) {
                __threadfence();
                if (lane == 0) P.unit_count[u] = 0;  // ready for the next launch
                if (hw == 0) {
                    // merge all pieces in segment order (deterministic), from L2
                    float M[G], L[G];
#pragma unroll
                    for (int h = 0; h < G; ++h) { M[h] = -INFINITY; L[h] = 0.f; }
                    const int base = P.unit_seg[u];
                    for (int sg = 0; sg < nseg; ++sg)
#pragma unroll
                        for (int h = 0; h < G; ++h)
                            M[h] = fmaxf(M[h], __ldcg(P.seg_ml + ((int64_t)(base + sg) * G + h) * 2));
#pragma unroll
                    for (int h = 0; h < G; ++h)
#pragma unroll
                        for (int i = 0; i < 4; ++i) o2[h][i] = make_float2(0.f, 0.f);
                    for (int sg = 0; sg < nseg; ++sg) {
#pragma unroll
                        for (int h = 0; h < G; ++h) {
                            const float2 ml = __ldcg(reinterpret_cast<const float2 *>(
                                P.seg_ml + ((int64_t)(base + sg) * G + h) * 2));
                            const float w = (ml.y > 0.f) ? ptx::ex2(ml.x - M[h]) : 0.f;
                            L[h] += ml.y * w;
                            const float4 *src = reinterpret_cast<const float4 *>(
                                P.seg_o + ((int64_t)(base + sg) * G + h) * D + c * 8);
                            const float4 x0 = __ldcg(src), x1 = __ldcg(src + 1);
                            const float2 ww = make_float2(w, w);
                            o2[h][0] = ptx::ffma2(ww, make_float2(x0.x, x0.y), o2[h][0]);
                            o2[h][1] = ptx::ffma2(ww, make_float2(x0.z, x0.w), o2[h][1]);
                            o2[h][2] = ptx::ffma2(ww, make_float2(x1.x, x1.y), o2[h][2]);
                            o2[h][3] = ptx::ffma2(ww, make_float2(x1.z, x1.w), o2[h][3]);
                        }
                    }
                    finalize<D, G>(a, req, head, c, M, L, o2);
                }
            }
        }
        __syncwarp();
    }
    }
    if (lane == 0 && atomicAdd(&P.sched[1], 1) == P.nwarps - 1) {  // last warp out: reset queues
        P.sched[1] = 0;
        for (int q = 0; q < kK2Queues; ++q) P.sched[2 + q] = 0;
    }
    K2_TRACE(2);
}

template <int D, int G>
cudaError_t launch_t(const SuffixArgs &a, int num_sms, cudaStream_t s) {
    using S = Shape<D, G>;
    const int smem = kWarps * S::WARP_SMEM_AL;
    auto kern = suffix_decode_kernel<D, G>;
    int dev = 0;
    cudaGetDevice(&dev);
    static bool configured[64] = {};  // the attribute is per function and device
    if (dev < 64 && !configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        configured[dev] = true;
    }
    if (a.p.nunits == 0) return cudaSuccess;
    const int grid = (a.p.nwarps + kWarps - 1) / kWarps;  // = num_sms: one CTA per SM
    kern<<<grid, kWarps * 32, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_suffix_decode(const PlanDev &p, const PoolGeom &g, const void *pool_k,
                                 const void *pool_v, int layer, const void *q, float *out,
                                 float *lse, float scale, int num_sms, cudaStream_t s) {
    SuffixArgs a;
    a.p = p;
    a.pool_k = static_cast<const uint16_t *>(pool_k);
    a.pool_v = static_cast<const uint16_t *>(pool_v);
    a.layer_off = (int64_t)layer * g.cap * g.hkv * kBlockTok * g.d;
    a.q = static_cast<const uint16_t *>(q);
    a.out = out;
    a.lse = lse;
    a.hkv = g.hkv;
    a.hq = g.hq;
    a.qscale = scale * kLog2e;
    static const int load_mode = [] {
        const char *e = getenv("HALO_K2_LOAD");
        return e ? atoi(e) : 0;
    }();
    a.load_mode = load_mode;
    const int G = g.hq / g.hkv;
#define HALO_K2_CASE(DD, GG) \
    if (g.d == DD && G == GG) return launch_t<DD, GG>(a, num_sms, s);
    HALO_K2_CASE(128, 1) HALO_K2_CASE(128, 2) HALO_K2_CASE(128, 4) HALO_K2_CASE(128, 8)
    HALO_K2_CASE(64, 1) HALO_K2_CASE(64, 2) HALO_K2_CASE(64, 4) HALO_K2_CASE(64, 8)
#undef HALO_K2_CASE
    return cudaErrorInvalidValue;
}

}  // namespace halo
