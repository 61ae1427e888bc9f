// K1: shared-prefix attention on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// What it computes: for one prefix node n (a shared segment of the consolidated query
// plan's prefix tree; the "shared prefix cache") and one
// kv head j, all decode queries of the requests under n form a dense matrix
//     Q_nj = [rows = (request under n) x (q-head of group j)] x d
// and the node's K/V are read ONCE for all of them:
//     S = Q_nj K_nj^T,   online softmax over the node's tokens,   O = P V_nj.
// Output: per (request, q-head) a normalised fp32 partial o and its natural-log lse, which
// K3 (fused into K2) merges with the private suffix -> identical to unshared attention
// ("Exact answers").
//
// Per CTA = one tile: 128 query rows (UMMA M) x a token range of the node (split-N).
//   warp 0      TMA producer: K/V tiles of 128 tokens = 8 paged 16-token blocks, one 4-D
//               TMA box per (block, 64-wide d atom), 128-B swizzle, 2-stage ring.
//   warp 1      MMA issuer (one thread): S_b = Q K^T into TMEM (double-buffered S0/S1),
//               O += P V into TMEM; tcgen05.commit -> mbarriers.
//   warp 2      TMEM allocator (512 columns: S0 | S1 | O).
//   warps 4..7  softmax warpgroup: thread i owns row i (TMEM lane i): tcgen05.ld of its
//               128 scores, row max / exp2 / row sum in registers (no shuffles), bf16 P
//               written to smem in the UMMA K-major SW128 layout, lazy O rescale (only
//               when the running max grows by > 2^8), final normalisation + store.
// Issue order QK(0) QK(1) PV(0) QK(2) PV(1) ... lets QK(n+1) run on the tensor pipe while
// the softmax warps work on S(n).
#include "halo_internal.h"
#include "ptx.h"

#include <cstdlib>

namespace halo {
namespace {

constexpr int kThreads = 256;
constexpr int kStagesKV = 2;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units: p <= 2^8 between rescales

struct PrefixArgs {
    PlanDev p;
    const uint16_t *q;  // [nreq][hq][D] bf16
    int32_t hq, hkv, g;
    int64_t layer_blk;  // layer * cap (4th TMA coordinate offset)
    float qscale;       // scale * log2(e)
};

template <int D>
struct L1 {
    static constexpr int ATOMS = D / 64;           // 128-B swizzle atoms along d
    static constexpr int ATOM_BYTES = 128 * 128;   // 128 rows x 128 B
    static constexpr int Q_BYTES = 128 * D * 2;
    static constexpr int KV_BYTES = kK1Tok * D * 2;
    static constexpr int P_BYTES = 128 * kK1Tok * 2;
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = OFF_Q + Q_BYTES;
    static constexpr int OFF_V = OFF_K + kStagesKV * KV_BYTES;
    static constexpr int OFF_P = OFF_V + kStagesKV * KV_BYTES;
    static constexpr int OFF_BAR = OFF_P + P_BYTES;
    static constexpr int NBAR = 16;
    static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;  // + alignment slack
    static constexpr int TMEM_S0 = 0, TMEM_S1 = 128, TMEM_O = 256;
};

enum Bar { Q_FULL = 0, K_FULL = 1, V_FULL = 3, KV_EMPTY = 5, S_FULL = 7, S_FREE = 9, P_FULL = 11,
           PV_DONE = 12, V_CONV = 13 };

// Precision of the P operand of O += P.V (reading R8):
//   kPBf16   bf16 P, bf16 V
//   kPMixed  fp16 P, bf16 V (A and B formats differ in the instruction descriptor)
//   kPF16    fp16 P, V converted bf16 -> fp16 in shared memory by warps 2-3
enum PMode { kPBf16 = 0, kPMixed = 1, kPF16 = 2 };

template <int D, int PM>
__global__ void __launch_bounds__(kThreads, 1)
prefix_attn_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                   const PrefixArgs a) {
    using C = L1<D>;
    extern __shared__ uint8_t smem_raw[];
    // 1024-B alignment for the 128-B swizzle atoms
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    uint8_t *sm = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + C::OFF_BAR);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + C::OFF_BAR + C::NBAR * 8);

    const PrefixTile T = a.p.tiles[blockIdx.x];
    const int NT = (T.tok_end - T.tok_begin + kK1Tok - 1) / kK1Tok;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar[Q_FULL], 128);
        for (int s = 0; s < kStagesKV; ++s) {
            ptx::mbar_init(&bar[K_FULL + s], 1);
            ptx::mbar_init(&bar[V_FULL + s], 1);
            ptx::mbar_init(&bar[KV_EMPTY + s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&bar[S_FULL + b], 1);
            ptx::mbar_init(&bar[S_FREE + b], 128);
        }
        ptx::mbar_init(&bar[P_FULL], 128);
        ptx::mbar_init(&bar[PV_DONE], 1);
        for (int s = 0; s < kStagesKV; ++s) ptx::mbar_init(&bar[V_CONV + s], 64);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc(tmem_slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            ptx::prefetch_tmap(&tmk);
            ptx::prefetch_tmap(&tmv);
            const int32_t *blocks = a.p.node_blocks + T.blk_off;
            for (int n = 0; n < NT; ++n) {
                const int st = n % kStagesKV;
                if (n >= kStagesKV) ptx::mbar_wait(&bar[KV_EMPTY + st], ((n / kStagesKV) & 1) ^ 1);
                const int tok0 = T.tok_begin + n * kK1Tok;
                const int ntok = min(kK1Tok, T.tok_end - tok0);
                const int nb = (ntok + kBlockTok - 1) / kBlockTok;
                const int blk0 = tok0 / kBlockTok;
                uint8_t *kdst = sm + C::OFF_K + st * C::KV_BYTES;
                uint8_t *vdst = sm + C::OFF_V + st * C::KV_BYTES;
                ptx::mbar_arrive_expect_tx(&bar[K_FULL + st], C::KV_BYTES);
                for (int bi = 0; bi < kK1Tok / kBlockTok; ++bi) {
                    // blocks past the tile's end re-load a valid block; their scores are masked
                    const int blk = blocks[blk0 + (bi < nb ? bi : 0)];
                    for (int at = 0; at < C::ATOMS; ++at)
                        ptx::tma_load_4d(kdst + at * C::ATOM_BYTES + bi * kBlockTok * 128, &tmk,
                                         at * 64, 0, T.kv_head, (int)(a.layer_blk + blk),
                                         &bar[K_FULL + st]);
                }
                ptx::mbar_arrive_expect_tx(&bar[V_FULL + st], C::KV_BYTES);
                for (int bi = 0; bi < kK1Tok / kBlockTok; ++bi) {
                    const int blk = blocks[blk0 + (bi < nb ? bi : 0)];
                    for (int at = 0; at < C::ATOMS; ++at)
                        ptx::tma_load_4d(vdst + at * C::ATOM_BYTES + bi * kBlockTok * 128, &tmv,
                                         at * 64, 0, T.kv_head, (int)(a.layer_blk + blk),
                                         &bar[V_FULL + st]);
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (single thread) =====================
        if (lane == 0) {
            constexpr uint32_t idS = ptx::idesc_bf16(128, kK1Tok, false, false);
            constexpr uint32_t idO = ptx::idesc_f16(128, D, PM == kPBf16 ? 1u : 0u,
                                                    PM == kPF16 ? 0u : 1u, false, true);
            const uint32_t q_base = ptx::smem_u32(sm + C::OFF_Q);
            const uint32_t p_base = ptx::smem_u32(sm + C::OFF_P);
            ptx::mbar_wait(&bar[Q_FULL], 0);
            ptx::tc_fence_after();
            for (int n = 0; n <= NT; ++n) {
                if (n < NT) {
                    const int st = n % kStagesKV, b = n & 1;
                    ptx::mbar_wait(&bar[K_FULL + st], (n / kStagesKV) & 1);
                    if (n >= 2) ptx::mbar_wait(&bar[S_FREE + b], ((n >> 1) & 1) ^ 1);
                    ptx::tc_fence_after();
                    const uint32_t k_base = ptx::smem_u32(sm + C::OFF_K + st * C::KV_BYTES);
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t off = (kk / 4) * C::ATOM_BYTES + (kk % 4) * 32;
                        ptx::mma_bf16_ss(tmem + (b ? C::TMEM_S1 : C::TMEM_S0),
                                         ptx::smem_desc_sw128(q_base + off, 16, 1024),
                                         ptx::smem_desc_sw128(k_base + off, 16, 1024), idS,
                                         kk > 0);
                    }
                    ptx::mma_commit(&bar[S_FULL + b]);
                }
                if (n >= 1) {
                    const int m = n - 1, st = m % kStagesKV;
                    if (PM == kPF16) ptx::mbar_wait(&bar[V_CONV + st], (m / kStagesKV) & 1);
                    else ptx::mbar_wait(&bar[V_FULL + st], (m / kStagesKV) & 1);
                    ptx::mbar_wait(&bar[P_FULL], m & 1);
                    ptx::tc_fence_after();
                    const uint32_t v_base = ptx::smem_u32(sm + C::OFF_V + st * C::KV_BYTES);
#pragma unroll
                    for (int kk = 0; kk < kK1Tok / 16; ++kk) {
                        const uint32_t aoff = (kk / 4) * C::ATOM_BYTES + (kk % 4) * 32;
                        // V as the MN-major B operand: 64-wide d chunks LBO = 128 rows x 128 B
                        // apart, 8-token row groups SBO = 1024 B apart; 16 tokens per step.
                        ptx::mma_bf16_ss(tmem + C::TMEM_O,
                                         ptx::smem_desc_sw128(p_base + aoff, 16, 1024),
                                         ptx::smem_desc_sw128(v_base + kk * 16 * 128, C::ATOM_BYTES, 1024),
                                         idO, (m > 0 || kk > 0) ? 1u : 0u);
                    }
                    ptx::mma_commit(&bar[KV_EMPTY + st]);
                    ptx::mma_commit(&bar[PV_DONE]);
                }
            }
        }
    } else if (PM == kPF16 && (warp == 2 || warp == 3)) {
        // ===================== V converter: bf16 -> fp16 in place =====================
        const int t = threadIdx.x - 64;  // 0..63
        for (int n = 0; n < NT; ++n) {
            const int st = n % kStagesKV;
            ptx::mbar_wait(&bar[V_FULL + st], (n / kStagesKV) & 1);
            uint4 *vs = reinterpret_cast<uint4 *>(sm + C::OFF_V + st * C::KV_BYTES);
#pragma unroll 4
            for (int c = t; c < C::KV_BYTES / 16; c += 64) {
                uint4 w = vs[c];
                float2 f;
                f = ptx::bf2_to_f2(w.x); w.x = ptx::f2_to_h2(f.x, f.y);
                f = ptx::bf2_to_f2(w.y); w.y = ptx::f2_to_h2(f.x, f.y);
                f = ptx::bf2_to_f2(w.z); w.z = ptx::f2_to_h2(f.x, f.y);
                f = ptx::bf2_to_f2(w.w); w.w = ptx::f2_to_h2(f.x, f.y);
                vs[c] = w;
            }
            ptx::fence_proxy_async_smem();
            ptx::mbar_arrive(&bar[V_CONV + st]);
        }
    } else if (warp >= 4) {
        // ===================== softmax warpgroup =====================
        const int r = threadIdx.x - 128;       // tile row == TMEM lane
        const int wq = warp - 4;
        const uint32_t lane_addr = tmem + ((uint32_t)(32 * wq) << 16);
        const bool valid_row = r < T.nrows;
        const int g = a.g;
        const int req = valid_row ? a.p.req_order[T.req_off + r / g] : 0;
        const int head = T.kv_head * g + r % g;
        // Q row -> smem, K-major SW128 (16-B chunk c of row r lands at chunk c ^ (r & 7))
        {
            const uint4 *src = reinterpret_cast<const uint4 *>(a.q + ((int64_t)req * a.hq + head) * D);
            uint8_t *qs = sm + C::OFF_Q;
#pragma unroll
            for (int c = 0; c < D / 8; ++c) {
                const uint4 v = valid_row ? src[c] : make_uint4(0, 0, 0, 0);
                const int at = c / 8, cc = c % 8;
                *reinterpret_cast<uint4 *>(qs + at * C::ATOM_BYTES + r * 128 + ((cc ^ (r & 7)) * 16)) = v;
            }
            ptx::fence_proxy_async_smem();
            ptx::mbar_arrive(&bar[Q_FULL]);
        }
        float m_ref = -INFINITY, l = 0.f;
        const float c2 = a.qscale;
        uint8_t *ps = sm + C::OFF_P;
        for (int n = 0; n < NT; ++n) {
            const int b = n & 1;
            ptx::mbar_wait(&bar[S_FULL + b], (n >> 1) & 1);
            ptx::tc_fence_after();
            uint32_t sr[kK1Tok];
#pragma unroll
            for (int k = 0; k < kK1Tok / 32; ++k) {
                uint32_t *dst = sr + 32 * k;
                HALO_TMEM_LD32(lane_addr + (b ? C::TMEM_S1 : C::TMEM_S0) + 32 * k, dst);
            }
            ptx::tmem_wait_ld();
            ptx::tc_fence_before();
            ptx::mbar_arrive(&bar[S_FREE + b]);

            const int valid = min(kK1Tok, T.tok_end - (T.tok_begin + n * kK1Tok));
            float mx = -INFINITY;
#pragma unroll
            for (int i = 0; i < kK1Tok; ++i)
                if (i < valid) mx = fmaxf(mx, __uint_as_float(sr[i]));
            const float mx2 = mx * c2;
            const bool grow = mx2 > m_ref + kRescaleThreshold;
            const float m_use = grow ? mx2 : m_ref;
            const float alpha = ptx::ex2(m_ref - m_use);  // 0 on the first tile
            uint32_t pk[kK1Tok / 2];
            float psum = 0.f;
#pragma unroll
            for (int i = 0; i < kK1Tok; i += 2) {
                const float p0 = (i < valid) ? ptx::ex2(fmaf(__uint_as_float(sr[i]), c2, -m_use)) : 0.f;
                const float p1 = (i + 1 < valid) ? ptx::ex2(fmaf(__uint_as_float(sr[i + 1]), c2, -m_use)) : 0.f;
                psum += p0 + p1;
                pk[i / 2] = PM == kPBf16 ? ptx::f2_to_bf2(p0, p1) : ptx::f2_to_h2(p0, p1);
            }
            l = l * alpha + psum;
            if (n >= 1) {
                ptx::mbar_wait(&bar[PV_DONE], (n - 1) & 1);  // P buffer free, O stable
                ptx::tc_fence_after();
                if (__any_sync(0xffffffffu, grow)) {
#pragma unroll
                    for (int k = 0; k < D / 32; ++k) {
                        uint32_t ov[32];
                        HALO_TMEM_LD32(lane_addr + C::TMEM_O + 32 * k, ov);
                        ptx::tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
                        HALO_TMEM_ST32(lane_addr + C::TMEM_O + 32 * k, ov);
                    }
                    ptx::tmem_wait_st();
                }
            }
            m_ref = m_use;
#pragma unroll
            for (int c = 0; c < kK1Tok / 8; ++c) {
                const int at = c / 8, cc = c % 8;
                *reinterpret_cast<uint4 *>(ps + at * C::ATOM_BYTES + r * 128 + ((cc ^ (r & 7)) * 16)) =
                    make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
            }
            ptx::fence_proxy_async_smem();
            ptx::tc_fence_before();
            ptx::mbar_arrive(&bar[P_FULL]);
        }
        // ---- epilogue: O / l -> normalised partial, lse ----
        ptx::mbar_wait(&bar[PV_DONE], (NT - 1) & 1);
        ptx::tc_fence_after();
        const float inv = 1.f / l;
        const int64_t row = ((int64_t)T.slot * a.p.nreq + req) * a.hq + head;
        float4 *dst = reinterpret_cast<float4 *>(a.p.part_o + row * D);
#pragma unroll
        for (int k = 0; k < D / 32; ++k) {
            uint32_t ov[32];
            HALO_TMEM_LD32(lane_addr + C::TMEM_O + 32 * k, ov);
            ptx::tmem_wait_ld();
            if (valid_row) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    dst[k * 8 + i] = make_float4(__uint_as_float(ov[4 * i]) * inv, __uint_as_float(ov[4 * i + 1]) * inv,
                                                 __uint_as_float(ov[4 * i + 2]) * inv, __uint_as_float(ov[4 * i + 3]) * inv);
            }
        }
        if (valid_row) a.p.part_lse[row] = (m_ref + __log2f(l)) * kLn2;
        ptx::tc_fence_before();
    }
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

template <int D, int PM>
cudaError_t launch_t(const CUtensorMap *tmk, const CUtensorMap *tmv, const PrefixArgs &a,
                     cudaStream_t s) {
    auto kern = prefix_attn_kernel<D, PM>;
    int dev = 0;
    cudaGetDevice(&dev);
    static bool configured[64] = {};
    if (dev < 64 && !configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L1<D>::SMEM);
        if (e != cudaSuccess) return e;
        configured[dev] = true;
    }
    kern<<<a.p.ntiles, kThreads, L1<D>::SMEM, s>>>(*tmk, *tmv, a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_prefix_attn(const CUtensorMap *tmap_k, const CUtensorMap *tmap_v,
                               const PlanDev &p, const PoolGeom &g, int layer, const void *q,
                               float scale, cudaStream_t s) {
    if (p.ntiles == 0) return cudaSuccess;
    PrefixArgs a;
    a.p = p;
    a.q = static_cast<const uint16_t *>(q);
    a.hq = g.hq;
    a.hkv = g.hkv;
    a.g = g.hq / g.hkv;
    a.layer_blk = (int64_t)layer * g.cap;
    a.qscale = scale * kLog2e;
    static const int pmode = [] {
        const char *e = getenv("HALO_K1_PMODE");
        return e ? atoi(e) : (int)kPF16;
    }();
#define HALO_K1_CASE(DD, PMM) \
    if (g.d == DD && pmode == PMM) return launch_t<DD, PMM>(tmap_k, tmap_v, a, s);
    HALO_K1_CASE(128, kPBf16) HALO_K1_CASE(128, kPMixed) HALO_K1_CASE(128, kPF16)
    HALO_K1_CASE(64, kPBf16) HALO_K1_CASE(64, kPMixed) HALO_K1_CASE(64, kPF16)
#undef HALO_K1_CASE
    return cudaErrorInvalidValue;
}

}  // namespace halo
