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
//  * warp-persistent streaming: every warp owns a ring of kStages smem stages and walks
//    work units (r, j) with a grid stride; its lane 0 issues one 1-D bulk async copy
//    (cp.async.bulk, TMA engine) per 4-KiB K slab and V slab of a 16-token block, with
//    completion on a per-stage mbarrier.  Prefetch runs ahead ACROSS unit boundaries, so
//    short suffixes do not drain the pipe.  Each K/V element is read from HBM once for
//    all g q-heads of its kv head (GQA reuse).
//  * compute from smem on CUDA cores: a token row is split over d/8 lanes (16-B LDS per
//    lane); q.k partial sums of the g heads are combined with a transpose-reduce
//    (log2(d/8)+g-1 shuffles instead of g*log2(d/8)), fp32x2 FMAs (FFMA2) for the dot
//    products and the P.V update, online softmax in base 2 with fp32 state.
//  * K3 epilogue: merge the suffix state with the normalised fp32 K1 partials of the
//    request (slots in a fixed order -> bit-deterministic), write fp32 out and lse.
#include "halo_internal.h"
#include "ptx.h"

namespace halo {
namespace {

constexpr int kWarps = 8;
constexpr int kStages = 3;
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
    static constexpr int WARP_SMEM = RING + PS + 16 * 4 + kStages * 8;
    static constexpr int WARP_SMEM_AL = (WARP_SMEM + 127) / 128 * 128;
    static_assert(G <= LPT, "transpose-reduce needs g <= d/8");
};

// Sum each of v[0..G) over the LPT lanes of a token group; afterwards lane c holds the
// full sum of head c / (LPT/G) in v[0].
template <int G, int LPT>
__device__ __forceinline__ float transpose_reduce(float (&v)[G], int c) {
    int n = G;
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
        n = half;
        mask >>= 1;
    }
#pragma unroll
    for (int m = LPT / G / 2; m >= 1; m >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], m);
    return v[0];
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

    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) ptx::mbar_init(&full[s], 1);
        ptx::fence_barrier_init();
    }
    __syncwarp();

    const PlanDev &P = a.p;
    const int hw = lane / S::LPT;   // token group within the warp
    const int c = lane % S::LPT;    // 16-B chunk of the row
    const int hsel = c / (S::LPT / G);
    const bool head_writer = (c % (S::LPT / G)) == 0;
    const int gw = blockIdx.x * kWarps + warp;
    const int nw = gridDim.x * kWarps;
    const uint16_t *pk = a.pool_k + a.layer_off;
    const uint16_t *pv = a.pool_v + a.layer_off;

    // ---- producer cursor (all lanes track it; lane 0 issues) ----
    int p_unit = gw, p_blk = 0, p_beg = 0, p_end = 0, p_head = 0;
    uint32_t p_count = 0, c_count = 0;
    auto load_unit = [&](int u, int &beg, int &end, int &head, int &req) {
        req = P.unit_req[u / a.hkv];
        head = u % a.hkv;
        beg = P.req_blk_off[req];
        end = P.req_blk_off[req + 1];
    };
    if (p_unit < P.nunits) {
        int req;
        load_unit(p_unit, p_beg, p_end, p_head, req);
    }
    auto fill = [&]() {
        while (p_unit < P.nunits && p_count - c_count < (uint32_t)kStages) {
            if (p_beg + p_blk < p_end) {
                if (lane == 0) {
                    const uint32_t e = P.req_blk[p_beg + p_blk];
                    const int64_t blk = e & kBlkMask;
                    const int64_t off = (blk * a.hkv + p_head) * (kBlockTok * D);
                    const int st = p_count % kStages;
                    uint8_t *dst = ws + st * S::STAGE;
                    ptx::mbar_arrive_expect_tx(&full[st], S::STAGE);
                    ptx::bulk_g2s(dst, pk + off, S::SLAB, &full[st]);
                    ptx::bulk_g2s(dst + S::SLAB, pv + off, S::SLAB, &full[st]);
                }
                ++p_blk;
                ++p_count;
            } else {
                p_unit += nw;
                p_blk = 0;
                if (p_unit < P.nunits) {
                    int req;
                    load_unit(p_unit, p_beg, p_end, p_head, req);
                }
            }
        }
    };
    fill();

    for (int u = gw; u < P.nunits; u += nw) {
        int beg, end, head, req;
        load_unit(u, beg, end, head, req);
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

        for (int b = beg; b < end; ++b) {
            fill();
            const int st = c_count % kStages;
            const int ntok = (int)(P.req_blk[b] >> kBlkCountShift) + 1;
            ptx::mbar_wait(&full[st], (c_count / kStages) & 1);
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
                    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc = ptx::ffma2(q2[h][i], ptx::bf2_to_f2(w[i]), acc);
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
        if (hw == 0) {
        // ---- K3: log-sum-exp merge with the prefix partials (base 2) ----
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
            const float ws_ = (lh[h] > 0.f) ? ptx::ex2(mh[h] - M[h]) : 0.f;
            L[h] = lh[h] * ws_;
#pragma unroll
            for (int i = 0; i < 4; ++i) o2[h][i] = ptx::fmul2(o2[h][i], make_float2(ws_, ws_));
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
        __syncwarp();
    }
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
    const int units_per_cta = kWarps;
    int grid = (a.p.nunits + units_per_cta - 1) / units_per_cta;
    if (grid > num_sms) grid = num_sms;  // 1 CTA (8 persistent warps) per SM
    if (grid < 1) return cudaSuccess;
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
    const int G = g.hq / g.hkv;
#define HALO_K2_CASE(DD, GG) \
    if (g.d == DD && G == GG) return launch_t<DD, GG>(a, num_sms, s);
    HALO_K2_CASE(128, 1) HALO_K2_CASE(128, 2) HALO_K2_CASE(128, 4) HALO_K2_CASE(128, 8)
    HALO_K2_CASE(64, 1) HALO_K2_CASE(64, 2) HALO_K2_CASE(64, 4) HALO_K2_CASE(64, 8)
#undef HALO_K2_CASE
    return cudaErrorInvalidValue;
}

}  // namespace halo
