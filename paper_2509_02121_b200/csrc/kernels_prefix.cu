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
//   warps 0-7   two softmax warpgroups; warp w owns TMEM lanes 32*(w%4).. (rows) and
//               column half w/4 of every S tile.  Each thread: thread i owns row i (TMEM lane i): tcgen05.ld of its
//               64 scores, row max (halves exchanged through smem), exp2 / row sum in
//               registers, P packed to 16-bit pairs and written to TMEM with tcgen05.st (no
//               smem traffic), lazy O rescale (only when the running max grows by > 2^8),
//               final normalisation.  Two warps per SMSP hide each other's latencies.
//   warp 8      TMA producer: two independent rings (K and V, 3 stages each); a 128-token
//               tile = 8 paged 16-token blocks, one 4-D TMA box per (block, 64-wide d atom),
//               128-B swizzle.  K stages free after Q.K^T, V stages after P.V.
//   warp 9      TMEM allocator (512 columns) + MMA issuer (one thread):
//               S_b = Q K^T (SS, double-buffered S0/S1), O += P V (A = P from TMEM).
//   warps 10-11 V converters (fp16-P mode): bf16 -> fp16 in place on each V stage, so the
//               P.V MMA runs with fp16 operands (P in fp16 is 8x more precise than bf16;
//               kind::f16 needs A and B in the same format).

// TMEM columns: S0 [0,128) | S1 [128,256) | O [256,256+d) | P0 [384,448) | P1 [448,512).
// Issue order QK(0) QK(1) PV(0) QK(2) PV(1) ... : QK(n+1) runs while softmax works on S(n).
#include "halo_internal.h"
#include "ptx.h"

#include <cstdlib>

#ifdef HALO_K1_TRACE
// Debug timeline of CTA 0: g_k1_trace[event * 64 + tile] = %globaltimer (ns).
__device__ unsigned long long *g_k1_trace = nullptr;  // [12][64]
#define K1_TRACE(ev, n)                                                                 \
    do {                                                                                \
        if (blockIdx.x == 0 && g_k1_trace && (n) < 64) {                                \
            unsigned long long t_;                                                      \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                    \
            g_k1_trace[(ev) * 64 + (n)] = t_;                                           \
        }                                                                               \
    } while (0)
extern "C" int halo_debug_k1_trace(void *buf) {
    return (int)cudaMemcpyToSymbol(g_k1_trace, &buf, sizeof(buf));
}
#else
#define K1_TRACE(ev, n) do { } while (0)
#endif

namespace halo {
namespace {

constexpr int kThreads = 384;  // 12 warps: 3 per SMSP (<= 168 registers per thread)
constexpr int kSoftmaxThreads = 256;
constexpr int kStagesKV = 3;
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
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_K = OFF_Q + Q_BYTES;
    static constexpr int OFF_V = OFF_K + kStagesKV * KV_BYTES;
    static constexpr int OFF_BAR = OFF_V + kStagesKV * KV_BYTES;
    static constexpr int NBAR = 24;
    static constexpr int OFF_BLK = OFF_BAR + NBAR * 8 + 16;       // block ids of the tile range
    static constexpr int MAX_BLK = kK1MaxTileTok / kBlockTok;    // block ids per CTA range
    static constexpr int OFF_X = OFF_BLK + MAX_BLK * 4;            // [2 tiles][2 halves][128] max
    static constexpr int SMEM = OFF_X + 2 * 2 * 128 * 4;            // base must be 1024-aligned
    static constexpr int O_STRIDE = D * 4;                       // epilogue staging row bytes
    static constexpr int TMEM_S0 = 0, TMEM_S1 = 128, TMEM_O = 256, TMEM_P = 384;
};

static_assert(L1<128>::SMEM <= 227 * 1024, "K1 shared memory exceeds the 227 KB per-CTA limit");

enum Bar {
    Q_FULL = 0,
    K_FULL = 1, K_EMPTY = 4, V_FULL = 7, V_EMPTY = 10, V_CONV = 13,  // x kStagesKV
    S_FULL = 16, S_FREE = 18, P_FULL = 20, PV_DONE = 22              // x 2
};

// Precision of the P operand of O += P.V (reading R8):
//   kPBf16   bf16 P, bf16 V (fails the 2e-3 bar on sharp score distributions)
//   kPF16    fp16 P, V converted bf16 -> fp16 in shared memory (default)
enum PMode { kPBf16 = 0, kPF16 = 2 };

template <int D, int PM>
__global__ void __launch_bounds__(kThreads, 1)
prefix_attn_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                   const __grid_constant__ CUtensorMap tmk8, const __grid_constant__ CUtensorMap tmv8,
                   const PrefixArgs a) {
    using C = L1<D>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 128-B swizzle atoms need a 1024-B aligned base (the dynamic window starts aligned)
    if (ptx::smem_u32(smem_raw) & 1023) __trap();
    uint8_t *sm = smem_raw;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + C::OFF_BAR);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + C::OFF_BAR + C::NBAR * 8);

    if (threadIdx.x == 0) K1_TRACE(9, 0);
    const PrefixTile T = a.p.tiles[blockIdx.x];
    const int NT = (T.tok_end - T.tok_begin + kK1Tok - 1) / kK1Tok;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar[Q_FULL], kSoftmaxThreads);
        for (int s = 0; s < kStagesKV; ++s) {
            ptx::mbar_init(&bar[K_FULL + s], 1);
            ptx::mbar_init(&bar[K_EMPTY + s], 1);
            ptx::mbar_init(&bar[V_FULL + s], 1);
            ptx::mbar_init(&bar[V_EMPTY + s], 1);
            ptx::mbar_init(&bar[V_CONV + s], 64);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&bar[S_FULL + b], 1);
            ptx::mbar_init(&bar[S_FREE + b], kSoftmaxThreads);
            ptx::mbar_init(&bar[P_FULL + b], kSoftmaxThreads);
            ptx::mbar_init(&bar[PV_DONE + b], 1);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 9) ptx::tmem_alloc(tmem_slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 8) {
        // ===================== TMA producer: K and V rings =====================
        // block ids of [tok_begin, tok_end) -> smem, all lanes, independent loads
        int32_t *blocks = reinterpret_cast<int32_t *>(sm + C::OFF_BLK);
        const int blk_first = T.tok_begin / kBlockTok;
        const int nblk = (T.tok_end + kBlockTok - 1) / kBlockTok - blk_first;
        for (int i = lane; i < nblk; i += 32) blocks[i] = a.p.node_blocks[T.blk_off + blk_first + i];
        __syncwarp();
        if (lane == 0) {
            ptx::prefetch_tmap(&tmk);
            ptx::prefetch_tmap(&tmv);
            ptx::prefetch_tmap(&tmk8);
            ptx::prefetch_tmap(&tmv8);
            auto issue = [&](const CUtensorMap *map, const CUtensorMap *map8, uint8_t *dst, uint64_t *full, int n) {
                const int tok0 = T.tok_begin + n * kK1Tok;
                const int nb = (min(kK1Tok, T.tok_end - tok0) + kBlockTok - 1) / kBlockTok;
                const int blk0 = tok0 / kBlockTok - blk_first;
                ptx::mbar_arrive_expect_tx(full, C::KV_BYTES);
                const int b0 = blocks[blk0];
                bool contiguous = nb == kK1Tok / kBlockTok;
#pragma unroll
                for (int bi = 1; bi < kK1Tok / kBlockTok; ++bi)
                    contiguous &= (bi >= nb) || blocks[blk0 + bi] == b0 + bi;
                if (contiguous) {  // physically consecutive blocks: one 128-token box per d atom
                    for (int at = 0; at < C::ATOMS; ++at)
                        ptx::tma_load_4d(dst + at * C::ATOM_BYTES, map8, at * 64, 0, T.kv_head,
                                         (int)(a.layer_blk + b0), full);
                    return;
                }
                for (int bi = 0; bi < kK1Tok / kBlockTok; ++bi) {
                    // blocks past the tile's end re-load a valid block; their scores are masked
                    const int blk = blocks[blk0 + (bi < nb ? bi : 0)];
                    for (int at = 0; at < C::ATOMS; ++at)
                        ptx::tma_load_4d(dst + at * C::ATOM_BYTES + bi * kBlockTok * 128, map,
                                         at * 64, 0, T.kv_head, (int)(a.layer_blk + blk), full);
                }
            };
            int nk = 0, nv = 0;
            while (nk < NT || nv < NT) {
                const int before = nk + nv;
                if (nk < NT && (nk < kStagesKV ||
                                ptx::mbar_test(&bar[K_EMPTY + nk % kStagesKV], ((nk / kStagesKV) & 1) ^ 1))) {
                    const int st = nk % kStagesKV;
                    issue(&tmk, &tmk8, sm + C::OFF_K + st * C::KV_BYTES, &bar[K_FULL + st], nk);
                    K1_TRACE(0, nk);
                    ++nk;
                }
                if (nv < NT && nv <= nk &&
                    (nv < kStagesKV ||
                     ptx::mbar_test(&bar[V_EMPTY + nv % kStagesKV], ((nv / kStagesKV) & 1) ^ 1))) {
                    const int st = nv % kStagesKV;
                    issue(&tmv, &tmv8, sm + C::OFF_V + st * C::KV_BYTES, &bar[V_FULL + st], nv);
                    K1_TRACE(1, nv);
                    ++nv;
                }
                if (nk + nv == before) __nanosleep(64);
            }
        }
    } else if (warp == 9) {
        // ===================== MMA issuer (single thread) =====================
        if (lane == 0) {
            constexpr uint32_t idS = ptx::idesc_bf16(128, kK1Tok, false, false);
            constexpr uint32_t fmtPV = PM == kPBf16 ? 1u : 0u;
            constexpr uint32_t idO = ptx::idesc_f16(128, D, fmtPV, fmtPV, false, true);
            const uint32_t q_base = ptx::smem_u32(sm + C::OFF_Q);
            ptx::mbar_wait(&bar[Q_FULL], 0);
            ptx::tc_fence_after();
            for (int n = 0; n <= NT; ++n) {
                if (n < NT) {
                    const int st = n % kStagesKV, b = n & 1;
                    ptx::mbar_wait(&bar[K_FULL + st], (n / kStagesKV) & 1);
                    if (n >= 2) ptx::mbar_wait(&bar[S_FREE + b], ((n >> 1) & 1) ^ 1);
                    K1_TRACE(2, n);
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
                    ptx::mma_commit(&bar[K_EMPTY + st]);
                }
                if (n >= 1) {
                    const int m = n - 1, st = m % kStagesKV, b = m & 1;
                    if (PM == kPF16) ptx::mbar_wait(&bar[V_CONV + st], (m / kStagesKV) & 1);
                    else ptx::mbar_wait(&bar[V_FULL + st], (m / kStagesKV) & 1);
                    ptx::mbar_wait(&bar[P_FULL + b], (m >> 1) & 1);
                    K1_TRACE(3, m);
                    ptx::tc_fence_after();
                    const uint32_t v_base = ptx::smem_u32(sm + C::OFF_V + st * C::KV_BYTES);
#pragma unroll
                    for (int kk = 0; kk < kK1Tok / 16; ++kk) {
                        // A = P from TMEM: 16 tokens = 8 packed 32-bit columns per K-step.
                        // B = V, MN-major: 64-wide d chunks LBO = 128 rows x 128 B apart,
                        // 8-token row groups SBO = 1024 B apart; 16 tokens per step.
                        ptx::mma_f16_ts(tmem + C::TMEM_O, tmem + C::TMEM_P + b * 64 + kk * 8,
                                        ptx::smem_desc_sw128(v_base + kk * 16 * 128, C::ATOM_BYTES, 1024),
                                        idO, (m > 0 || kk > 0) ? 1u : 0u);
                    }
                    ptx::mma_commit(&bar[V_EMPTY + st]);
                    ptx::mma_commit(&bar[PV_DONE + b]);
                }
            }
        }
    } else if (warp >= 10) {
        // ===================== V converters: bf16 -> fp16 in place =====================
        if (PM == kPF16) {
            const int t = threadIdx.x - 320;  // 0..63
            for (int n = 0; n < NT; ++n) {
                const int st = n % kStagesKV;
                ptx::mbar_wait(&bar[V_FULL + st], (n / kStagesKV) & 1);
                if (t == 0) K1_TRACE(4, n);
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
                if (t == 0) K1_TRACE(5, n);
                ptx::mbar_arrive(&bar[V_CONV + st]);
            }
        }
    } else {
        // ===================== softmax warpgroups (warps 0..7) =====================
        constexpr int HC = kK1Tok / 2;          // columns per half
        const int h = warp >> 2;                // column half
        const int wq = warp & 3;
        const int r = wq * 32 + lane;           // tile row == TMEM lane
        const int st_id = threadIdx.x;          // 0..255
        const uint32_t lane_addr = tmem + ((uint32_t)(32 * wq) << 16);
        const bool valid_row = r < T.nrows;
        const int g = a.g;
        const int req = valid_row ? a.p.req_order[T.req_off + r / g] : 0;
        const int head = T.kv_head * g + r % g;
        float *xmax = reinterpret_cast<float *>(sm + C::OFF_X);  // [2][2][128]
        // Q row -> smem, K-major SW128 (16-B chunk c of row r lands at chunk c ^ (r & 7));
        // each half loads half of the row's chunks
        {
            const uint4 *src = reinterpret_cast<const uint4 *>(a.q + ((int64_t)req * a.hq + head) * D);
            uint8_t *qs = sm + C::OFF_Q;
#pragma unroll
            for (int cc0 = 0; cc0 < D / 16; ++cc0) {
                const int c = h * (D / 16) + cc0;
                const uint4 v = valid_row ? src[c] : make_uint4(0, 0, 0, 0);
                const int at = c / 8, cc = c % 8;
                *reinterpret_cast<uint4 *>(qs + at * C::ATOM_BYTES + r * 128 + ((cc ^ (r & 7)) * 16)) = v;
            }
            ptx::fence_proxy_async_smem();
            if (st_id == 0) K1_TRACE(9, 2);
            ptx::mbar_arrive(&bar[Q_FULL]);
        }
        float m_ref = -INFINITY, l = 0.f;
        const float c2 = a.qscale;
        for (int n = 0; n < NT; ++n) {
            const int b = n & 1;
            ptx::mbar_wait(&bar[S_FULL + b], (n >> 1) & 1);
            if (st_id == 0) K1_TRACE(6, n);
            ptx::tc_fence_after();
            const uint32_t s_addr = lane_addr + (b ? C::TMEM_S1 : C::TMEM_S0) + h * HC;
            const int valid = min(kK1Tok, T.tok_end - (T.tok_begin + n * kK1Tok)) - h * HC;
            uint32_t sr[HC];
            HALO_TMEM_LD32(s_addr, sr);
            HALO_TMEM_LD32(s_addr + 32, (sr + 32));
            ptx::tmem_wait_ld();
            ptx::tc_fence_before();
            ptx::mbar_arrive(&bar[S_FREE + b]);
            if (valid < HC) {  // only in a node's last tile: columns past the end -> -inf
#pragma unroll
                for (int i = 0; i < HC; ++i)
                    if (i >= valid) sr[i] = __float_as_uint(-INFINITY);
            }
            float mxv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) mxv[i] = __uint_as_float(sr[i]);
#pragma unroll
            for (int i = 8; i < HC; ++i) mxv[i & 7] = fmaxf(mxv[i & 7], __uint_as_float(sr[i]));
            float mx = fmaxf(fmaxf(fmaxf(mxv[0], mxv[1]), fmaxf(mxv[2], mxv[3])),
                             fmaxf(fmaxf(mxv[4], mxv[5]), fmaxf(mxv[6], mxv[7])));
            // exchange the half-row maxima (double-buffered by tile parity)
            xmax[(b * 2 + h) * 128 + r] = mx;
            asm volatile("bar.sync 1, 256;" ::: "memory");
            mx = fmaxf(mx, xmax[(b * 2 + (h ^ 1)) * 128 + r]);
            if (st_id == 0) K1_TRACE(7, n);
            const float mx2 = mx * c2;
            const bool grow = mx2 > m_ref + kRescaleThreshold;
            const float m_use = grow ? mx2 : m_ref;
            const float alpha = ptx::ex2(m_ref - m_use);  // 0 on the first tile
            if (n >= 2) ptx::mbar_wait(&bar[PV_DONE + b], ((n >> 1) - 1) & 1);  // P[b] consumed
            if (n >= 1 && __any_sync(0xffffffffu, grow)) {
                ptx::mbar_wait(&bar[PV_DONE + (b ^ 1)], ((n - 1) >> 1) & 1);  // O stable
                ptx::tc_fence_after();
#pragma unroll
                for (int k = 0; k < D / 64; ++k) {
                    uint32_t ov[32];
                    const uint32_t oa = lane_addr + C::TMEM_O + h * (D / 2) + 32 * k;
                    HALO_TMEM_LD32(oa, ov);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
                    HALO_TMEM_ST32(oa, ov);
                }
            }
            m_ref = m_use;
            ptx::tc_fence_after();
            if (st_id == 0) K1_TRACE(10, n);
            // p = 2^(s*c - m) (masked scores give 0), packed 16-bit pairs -> TMEM P[b]
            const float2 c2v = make_float2(c2, c2), nm = make_float2(-m_use, -m_use);
            float2 psv[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
            for (int k = 0; k < HC / 32; ++k) {
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
                    const int col = 32 * k + i;
                    float2 x = ptx::ffma2(make_float2(__uint_as_float(sr[col]), __uint_as_float(sr[col + 1])), c2v, nm);
                    x.x = ptx::ex2(x.x);
                    x.y = ptx::ex2(x.y);
                    psv[(i >> 1) & 1] = ptx::fadd2(psv[(i >> 1) & 1], x);
                    pk[i / 2] = PM == kPBf16 ? ptx::f2_to_bf2(x.x, x.y) : ptx::f2_to_h2(x.x, x.y);
                }
                HALO_TMEM_ST16(lane_addr + C::TMEM_P + b * 64 + h * (HC / 2) + 16 * k, pk);
            }
            if (st_id == 0) K1_TRACE(11, n);
            l = l * alpha + ((psv[0].x + psv[0].y) + (psv[1].x + psv[1].y));
            ptx::tmem_wait_st();
            if (st_id == 0) K1_TRACE(8, n);
            ptx::tc_fence_before();
            ptx::mbar_arrive(&bar[P_FULL + b]);
        }
        // ---- epilogue: O / l -> normalised partial, lse ----
        ptx::mbar_wait(&bar[PV_DONE + ((NT - 1) & 1)], ((NT - 1) >> 1) & 1);
        ptx::tc_fence_after();
        xmax[h * 128 + r] = l;  // row sums of the two halves (same reference max)
        asm volatile("bar.sync 1, 256;" ::: "memory");
        l += xmax[(h ^ 1) * 128 + r];
        const float inv = 1.f / l;
        // row r, this half's d columns -> smem staging (16-B chunks XOR-swizzled by row)
        uint8_t *stage = sm + C::OFF_K;  // K ring is free once the last PV completed
#pragma unroll
        for (int k = 0; k < D / 64; ++k) {
            uint32_t ov[32];
            HALO_TMEM_LD32(lane_addr + C::TMEM_O + h * (D / 2) + 32 * k, ov);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int c = h * (D / 8) + k * 8 + i;
                *reinterpret_cast<float4 *>(stage + r * C::O_STRIDE + ((c ^ (r & 7)) * 16)) =
                    make_float4(__uint_as_float(ov[4 * i]) * inv, __uint_as_float(ov[4 * i + 1]) * inv,
                                __uint_as_float(ov[4 * i + 2]) * inv, __uint_as_float(ov[4 * i + 3]) * inv);
            }
        }
        const int64_t row = ((int64_t)T.slot * a.p.nreq + req) * a.hq + head;
        int64_t *row_off = reinterpret_cast<int64_t *>(sm + C::OFF_V);  // V ring is free too
        if (h == 0) row_off[r] = valid_row ? row * D : -1;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        // each warp writes whole rows: lane = 16-B chunk (d=128: 32 chunks = 512 B per row)
        constexpr int CPR = D / 4;
        constexpr int RPI = 32 / CPR;  // rows per warp instruction
        for (int rr = warp * RPI; rr < 128; rr += 8 * RPI) {
            const int row_i = rr + lane / CPR, c = lane % CPR;
            const int64_t off = row_off[row_i];
            if (off >= 0)
                reinterpret_cast<float4 *>(a.p.part_o + off)[c] =
                    *reinterpret_cast<const float4 *>(stage + row_i * C::O_STRIDE + ((c ^ (row_i & 7)) * 16));
        }
        if (valid_row && h == 0) a.p.part_lse[row] = (m_ref + __log2f(l)) * kLn2;
        if (st_id == 0) K1_TRACE(9, 1);
        ptx::tc_fence_before();
    }
    __syncthreads();
    if (warp == 9) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

template <int D, int PM>
cudaError_t launch_t(const CUtensorMap *tmk, const CUtensorMap *tmv, const CUtensorMap *tmk8,
                     const CUtensorMap *tmv8, const PrefixArgs &a, cudaStream_t s) {
    auto kern = prefix_attn_kernel<D, PM>;
    int dev = 0;
    cudaGetDevice(&dev);
    static bool configured[64] = {};
    if (dev < 64 && !configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L1<D>::SMEM);
        if (e != cudaSuccess) return e;
        configured[dev] = true;
    }
    kern<<<a.p.ntiles, kThreads, L1<D>::SMEM, s>>>(*tmk, *tmv, *tmk8, *tmv8, a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_prefix_attn(const CUtensorMap *tmap_k, const CUtensorMap *tmap_v,
                               const CUtensorMap *tmap_k8, const CUtensorMap *tmap_v8,
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
    if (g.d == DD && pmode == PMM) return launch_t<DD, PMM>(tmap_k, tmap_v, tmap_k8, tmap_v8, a, s);
    HALO_K1_CASE(128, kPBf16) HALO_K1_CASE(128, kPF16)
    HALO_K1_CASE(64, kPBf16) HALO_K1_CASE(64, kPF16)
#undef HALO_K1_CASE
    return cudaErrorInvalidValue;
}

}  // namespace halo
