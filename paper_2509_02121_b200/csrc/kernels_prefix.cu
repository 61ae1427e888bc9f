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
// Per CTA = one tile: 256 query rows as two UMMA M=128 sub-tiles A and B sharing every K/V
// stage (half the smem/TMA traffic per FLOP of a 128-row tile), x a token range of the
// node (split-N), 128-token n-tiles.
//   warps 0-3   softmax warpgroup A, warps 4-7 softmax warpgroup B: thread = one query row
//               of its sub-tile (= its TMEM lane), the full 128-column score row per n-tile,
//               so row max / row sum need no cross-thread exchange.  Online softmax in base
//               2 with a lazy reference max: p = 2^(s*c - m_ref) is computed optimistically
//               with the current m_ref (packed to fp16 pairs in registers) and only if some
//               row's max exceeds m_ref + 8 does the warp rescale O in TMEM and redo the
//               tile.  P is written with tcgen05.st over the sub-tile's own S columns.
//   warp 8      TMA producer: K ring (kSK stages) and V ring (kSV stages) of 128-token tiles
//               = 8 paged 16-token blocks (one 4-D box per 128-token run of physically
//               consecutive blocks, else one per block), 128-B swizzle.
//   warp 9      TMEM allocator (512 columns) + MMA issuer (one thread), ping-pong order
//                  PV_A(n-1) QK_A(n) PV_B(n-1) QK_B(n)
//               so softmax A(n) overlaps PV_B(n-1) + QK_B(n) on the tensor pipe and vice
//               versa.  tcgen05.mma executes in issue order, so QK_X(n) may overwrite the
//               S/P columns PV_X(n-1) reads.
//   warps 10-11 V converters: bf16 -> fp16 in place on each V stage (fp16 P needs fp16 V:
//               kind::f16 takes A and B in one format; reading R8), scaled by an
//               exact power of two 2^-s per tile so that any finite bf16 V fits fp16's range.
//               s comes from the pool's V table (max |V| per (layer, block), maintained by
//               every kernel that writes pool blocks): s = 0 while the tile's max |V| is in
//               [2^-4, 2^15), else (exponent of max) - 14, so converted values stay < 2^15 and
//               those >= max * 2^-29 stay fp16-normal; the epilogue multiplies by 2^s.  Powers of
//               two are exact: for in-range V nothing changes (K1, "V range").
//
// TMEM columns: S_A/P_A [0,128) | S_B/P_B [128,256) | O_A [256,256+d) | O_B [384,384+d).
#include "halo_internal.h"
#include "ptx.h"

#include <cuda_bf16.h>
#include <cstdlib>

#ifdef HALO_K1_TRACE
// Debug timeline of CTA 0: g_k1_trace[event * 64 + tile] = %globaltimer (ns).
__device__ unsigned long long *g_k1_trace = nullptr;  // [24][64]
#define K1_TRACE(ev, n)                                                                 \
    do {                                                                                \
        if (blockIdx.x == 0 && g_k1_trace && (n) < 64) {                                \
            unsigned long long t_;                                                      \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                    \
            g_k1_trace[(ev) * 64 + (n)] = t_;                                           \
        }                                                                               \
    } while (0)
// same, recorded only once `dep` has been computed (the timer read takes it as an operand)
#define K1_TRACE_DEP(ev, n, dep)                                                        \
    do {                                                                                \
        if (blockIdx.x == 0 && g_k1_trace && (n) < 64) {                                \
            unsigned long long t_;                                                      \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_) : "f"(dep));          \
            g_k1_trace[(ev) * 64 + (n)] = t_;                                           \
        }                                                                               \
    } while (0)
extern "C" int halo_debug_k1_trace(void *buf) {
    return (int)cudaMemcpyToSymbol(g_k1_trace, &buf, sizeof(buf));
}
#else
#define K1_TRACE(ev, n) do { } while (0)
#define K1_TRACE_DEP(ev, n, dep) do { } while (0)
#endif

#ifndef HALO_K1_PINGPONG
// MUFU ping-pong between the sub-tiles' exp passes: 1 = strict A/B alternation, 0 = none
// (default: C3 0.55 -> 0.56, C2 root 0.450 -> 0.457; profiles/k1_pingpong_ab_r02.txt)
#define HALO_K1_PINGPONG 0
#endif

namespace halo {
namespace {

constexpr int kThreads = 384;  // 12 warps: 3 per SMSP (<= 168 registers per thread)
constexpr int kSubRows = 128;  // rows per sub-tile (UMMA M)
constexpr int kRegsSoftmax = 208, kRegsOther = 88;  // 8 x 208 + 4 x 88 warps = 12 x 168
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units: p <= 2^8 between rescales
static_assert(kK1Rows == 2 * kSubRows, "K1 tile = two UMMA M=128 sub-tiles");

struct PrefixArgs {
    PlanDev p;
    const uint16_t *q;  // [nreq][hq][D] bf16
    int32_t hq, hkv, g;
    int64_t layer_blk;  // layer * cap (4th TMA coordinate offset)
    float qscale;       // scale * log2(e)
    int32_t tma_q;      // tmq is valid: tiles with consecutive requests load Q by TMA
    const uint64_t *vmax;  // the pool's V table [layer][block] (low 16 bits: bf16 max |V|)
    int64_t cap;
    int32_t layer;
};

template <int D>
struct L1 {
    static constexpr int SK = D == 128 ? 3 : 4;    // K ring stages
    static constexpr int SV = D == 128 ? 2 : 4;    // V ring stages
    static constexpr int ATOMS = D / 64;           // 128-B swizzle atoms along d
    static constexpr int ATOM_BYTES = 128 * 128;   // 128 rows x 128 B
    static constexpr int Q_BYTES = kSubRows * D * 2;   // one sub-tile
    static constexpr int KV_BYTES = kK1Tok * D * 2;
    static constexpr int OFF_Q = 0;                      // Q_A | Q_B
    static constexpr int OFF_K = OFF_Q + 2 * Q_BYTES;
    static constexpr int OFF_V = OFF_K + SK * KV_BYTES;
    static constexpr int OFF_BAR = OFF_V + SV * KV_BYTES;
    static constexpr int NBAR = 40;
    static constexpr int OFF_BLK = OFF_BAR + NBAR * 8 + 16;       // block ids of the tile range
    static constexpr int MAX_BLK = kK1MaxTileTok / kBlockTok;
    static constexpr int OFF_VEXP = OFF_BLK + MAX_BLK * 4;          // the tile's V scale exponent
    static constexpr int OFF_VRED = OFF_VEXP + 4 * 4;               // [2 warps] V max reduction
    static constexpr int SMEM = OFF_VRED + 4 * 4;                   // base must be 1024-aligned
    static constexpr int O_STRIDE = D * 4;                          // epilogue staging row bytes
    static __host__ __device__ constexpr uint32_t tmem_s(int x) { return x ? 128u : 0u; }
    static __host__ __device__ constexpr uint32_t tmem_o(int x) { return x ? 384u : 256u; }
    static_assert(SK * KV_BYTES >= kSubRows * O_STRIDE && SV * KV_BYTES >= kSubRows * O_STRIDE,
                  "epilogue staging reuses the K ring (A) and the V ring (B)");
    static_assert(SMEM <= 227 * 1024, "K1 shared memory exceeds the 227 KB per-CTA limit");
};

enum Bar {
    Q_FULL = 0,                                  // x2 (sub-tile)
    S_FULL = 2, P_FULL = 4, PV_DONE = 6,         // x2
    K_FULL = 8, K_EMPTY = 12,                    // x SK (<= 4)
    V_FULL = 16, V_EMPTY = 20, V_CONV = 24,      // x SV (<= 4)
    EXP_DONE = 28,                               // x8: warp (x, w) of sub-tile x finished its exp
                                                 // pass; index EXP_DONE + 4 x + w (w = warp & 3)

};

// TMA loads of n-tile n of tile T (128 tokens = 8 paged blocks) of K or V into `dst`, completing
// on `full` (expect_tx armed here): one 4-D box per d atom when the 8 blocks are physically
// consecutive, else one per block; blocks past the tile's end re-load a valid block (their
// scores are masked).  blocks = the tile's block ids from blk_first on (smem).
template <int D>
__device__ __forceinline__ void issue_kv_tile(const CUtensorMap *map, const CUtensorMap *map8, uint8_t *dst,
                                              uint64_t *full, const int32_t *blocks, const PrefixTile &T,
                                              int blk_first, int n, int64_t layer_blk) {
    using C = L1<D>;
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
            ptx::tma_load_4d(dst + at * C::ATOM_BYTES, map8, at * 64, 0, T.kv_head, (int)(layer_blk + b0), full);
        return;
    }
    for (int bi = 0; bi < kK1Tok / kBlockTok; ++bi) {
        const int blk = blocks[blk0 + (bi < nb ? bi : 0)];
        for (int at = 0; at < C::ATOMS; ++at)
            ptx::tma_load_4d(dst + at * C::ATOM_BYTES + bi * kBlockTok * 128, map, at * 64, 0, T.kv_head,
                             (int)(layer_blk + blk), full);
    }
}

// bf16 pair -> fp16 pair scaled by sc (an exact power of two; unit: no multiply).  satfinite:
// stale values in the masked tail of a suffix block can never become inf (P = 0 there, and
// 0 x inf would be nan).
__device__ __forceinline__ uint32_t cvt_v2(uint32_t w, float2 scv, bool unit) {
    float2 f = ptx::bf2_to_f2(w);
    if (!unit) f = ptx::fmul2(f, scv);
    uint32_t r;
    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(f.y), "f"(f.x));
    return r;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
prefix_attn_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                   const __grid_constant__ CUtensorMap tmk8, const __grid_constant__ CUtensorMap tmv8,
                   const __grid_constant__ CUtensorMap tmq, const PrefixArgs a) {
    using C = L1<D>;
    constexpr int SK = C::SK, SV = C::SV;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 128-B swizzle atoms need a 1024-B aligned base (the dynamic window starts aligned)
    if (ptx::smem_u32(smem_raw) & 1023) __trap();
    uint8_t *sm = smem_raw;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + C::OFF_BAR);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + C::OFF_BAR + C::NBAR * 8);

    if (threadIdx.x == 0) K1_TRACE(9, 0);
    // PDL: let K2 (the next kernel: streams private suffixes, reads our partials only after
    // griddepcontrol.wait) start on SMs this grid leaves idle and as its CTAs retire
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const PrefixTile T = a.p.tiles[blockIdx.x];
    const int4 aux = a.p.tile_aux[blockIdx.x];  // loaded alongside T (no dependency)
    const int NT = (T.tok_end - T.tok_begin + kK1Tok - 1) / kK1Tok;
    const bool hasB = T.nrows > kSubRows;
    // Q by TMA when the tile's requests are consecutive caller indices: one 3-D box
    // {64 d, g heads, 128/g requests} per sub-tile and d atom lands rows request-major, head
    // minor = the tile's row order, in the same 128-B swizzle the MMA descriptors expect
    const bool tma_q = a.tma_q && aux.x >= 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int x = 0; x < 2; ++x) {
            ptx::mbar_init(&bar[Q_FULL + x], tma_q ? 1 : kSubRows);
            ptx::mbar_init(&bar[S_FULL + x], 1);
            ptx::mbar_init(&bar[P_FULL + x], kSubRows);
            ptx::mbar_init(&bar[PV_DONE + x], 1);
            for (int w = 0; w < 4; ++w) ptx::mbar_init(&bar[EXP_DONE + 4 * x + w], 32);
        }
        for (int s = 0; s < SK; ++s) {
            ptx::mbar_init(&bar[K_FULL + s], 1);
            ptx::mbar_init(&bar[K_EMPTY + s], 1);
        }
        for (int s = 0; s < SV; ++s) {
            ptx::mbar_init(&bar[V_FULL + s], 1);
            ptx::mbar_init(&bar[V_EMPTY + s], 1);
            ptx::mbar_init(&bar[V_CONV + s], 64);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 9) ptx::tmem_alloc(tmem_slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) K1_TRACE(9, 3);  // barriers + TMEM allocated

    // register split (setmaxnreg, per warpgroup): the softmax warpgroups hold a full
    // 128-column score row per thread; the producer / MMA / converter warpgroup gives back
#define HALO_REGS_DEC() asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsOther))
#define HALO_REGS_INC() asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsSoftmax))
    if (warp == 8) {
        HALO_REGS_DEC();
        // ===================== TMA producer: K and V rings =====================
        int32_t *blocks = reinterpret_cast<int32_t *>(sm + C::OFF_BLK);
        const int blk_first = T.tok_begin / kBlockTok;
        const int nblk = (T.tok_end + kBlockTok - 1) / kBlockTok - blk_first;
        if (aux.y >= 0) {  // consecutive blocks: ids follow from the first (no global load)
            for (int i = lane; i < nblk; i += 32) blocks[i] = aux.y + i;
        } else {
            for (int i = lane; i < nblk; i += 32) blocks[i] = a.p.node_blocks[T.blk_off + blk_first + i];
        }
        __syncwarp();
        if (lane == 0) {  // descriptors are kernel parameters: fetch them before the wait
            ptx::prefetch_tmap(&tmk);
            ptx::prefetch_tmap(&tmv);
            ptx::prefetch_tmap(&tmk8);
            ptx::prefetch_tmap(&tmv8);
            if (tma_q) ptx::prefetch_tmap(&tmq);
        }
        // PDL: this grid may start while the previous kernel drains; the pool blocks it reads
        // may have been written by that kernel (a registration or append), so wait here
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (lane == 0) K1_TRACE(9, 4);  // producer: previous grid complete
        if (lane == 0) {
            if (tma_q) {
                const int rq = kSubRows / a.g;  // requests per sub-tile
                for (int x = 0; x < (hasB ? 2 : 1); ++x) {
                    ptx::mbar_arrive_expect_tx(&bar[Q_FULL + x], C::Q_BYTES);
                    for (int at = 0; at < C::ATOMS; ++at)
                        ptx::tma_load_3d(sm + C::OFF_Q + x * C::Q_BYTES + at * C::ATOM_BYTES, &tmq, at * 64,
                                         T.kv_head * a.g, aux.x + x * rq, &bar[Q_FULL + x]);
                }
            }
            auto issue = [&](const CUtensorMap *map, const CUtensorMap *map8, uint8_t *dst, uint64_t *full, int n) {
                issue_kv_tile<D>(map, map8, dst, full, blocks, T, blk_first, n, a.layer_blk);
            };
            int nk = 0, nv = 0;
            while (nk < NT || nv < NT) {
                const int before = nk + nv;
                if (nk < NT && (nk < SK || ptx::mbar_test(&bar[K_EMPTY + nk % SK], ((nk / SK) & 1) ^ 1))) {
                    issue(&tmk, &tmk8, sm + C::OFF_K + (nk % SK) * C::KV_BYTES, &bar[K_FULL + nk % SK], nk);
                    K1_TRACE(0, nk);
                    ++nk;
                }
                if (nv < NT && nv <= nk &&
                    (nv < SV || ptx::mbar_test(&bar[V_EMPTY + nv % SV], ((nv / SV) & 1) ^ 1))) {
                    issue(&tmv, &tmv8, sm + C::OFF_V + (nv % SV) * C::KV_BYTES, &bar[V_FULL + nv % SV], nv);
                    K1_TRACE(1, nv);
                    ++nv;
                }
                if (nk + nv == before) __nanosleep(32);
            }
        }
    } else if (warp == 9) {
        HALO_REGS_DEC();
        // ===================== MMA issuer (single thread) =====================
        if (lane == 0) {
            constexpr uint32_t idS = ptx::idesc_bf16(128, kK1Tok, false, false);
            constexpr uint32_t idO = ptx::idesc_f16(128, D, 0u, 0u, false, true);
            const int nsub = hasB ? 2 : 1;
            for (int x = 0; x < nsub; ++x) ptx::mbar_wait(&bar[Q_FULL + x], 0);
            ptx::tc_fence_after();
            for (int n = 0; n <= NT; ++n) {
                const int m = n - 1, vst = (m + SV) % SV, kst = n % SK;
                if (n < NT) {
                    ptx::mbar_wait(&bar[K_FULL + kst], (n / SK) & 1);
                    K1_TRACE(2, n);
                }
                if (n >= 1) {
                    ptx::mbar_wait(&bar[V_CONV + vst], (m / SV) & 1);
                    K1_TRACE(12, m);
                }
                for (int x = 0; x < nsub; ++x) {
                    if (n >= 1) {  // PV_x(m): A = P_x from TMEM (8 packed columns per 16 tokens)
                        ptx::mbar_wait(&bar[P_FULL + x], m & 1);
                        K1_TRACE(3 + 12 * x, m);
                        ptx::tc_fence_after();
                        const uint32_t v_base = ptx::smem_u32(sm + C::OFF_V + vst * C::KV_BYTES);
#pragma unroll
                        for (int kk = 0; kk < kK1Tok / 16; ++kk)
                            // B = V, MN-major: 64-wide d chunks LBO = 128 rows x 128 B apart,
                            // 8-token row groups SBO = 1024 B apart; 16 tokens per step.
                            ptx::mma_f16_ts(tmem + C::tmem_o(x), tmem + C::tmem_s(x) + kk * 8,
                                            ptx::smem_desc_sw128(v_base + kk * 16 * 128, C::ATOM_BYTES, 1024),
                                            idO, (m > 0 || kk > 0) ? 1u : 0u);
                        ptx::mma_commit(&bar[PV_DONE + x]);
                        if (x == nsub - 1) ptx::mma_commit(&bar[V_EMPTY + vst]);
                    }
                    if (n < NT) {  // QK_x(n) -> S_x (overwrites P_x(m): PV_x(m) was issued first)
                        const uint32_t q_base = ptx::smem_u32(sm + C::OFF_Q + x * C::Q_BYTES);
                        const uint32_t k_base = ptx::smem_u32(sm + C::OFF_K + kst * C::KV_BYTES);
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {
                            const uint32_t off = (kk / 4) * C::ATOM_BYTES + (kk % 4) * 32;
                            ptx::mma_bf16_ss(tmem + C::tmem_s(x), ptx::smem_desc_sw128(q_base + off, 16, 1024),
                                             ptx::smem_desc_sw128(k_base + off, 16, 1024), idS, kk > 0);
                        }
                        ptx::mma_commit(&bar[S_FULL + x]);
                        if (x == nsub - 1) ptx::mma_commit(&bar[K_EMPTY + kst]);
                    }
                }
            }
        }
    } else if (warp >= 10) {
        HALO_REGS_DEC();
        // ===================== V converters: bf16 -> fp16 in place, scaled =====================
        const int t = threadIdx.x - 320;  // 0..63
        int32_t *vexp = reinterpret_cast<int32_t *>(sm + C::OFF_VEXP);
        uint32_t *vred = reinterpret_cast<uint32_t *>(sm + C::OFF_VRED);
        // the tile's scale: max over its blocks' V-table entries (written by earlier kernels)
        asm volatile("griddepcontrol.wait;" ::: "memory");
        {
            const int blk_first = T.tok_begin / kBlockTok;
            const int nblk = (T.tok_end + kBlockTok - 1) / kBlockTok - blk_first;
            const uint64_t *vrow = a.vmax + (a.layer_blk / a.cap) * a.cap;
            uint32_t mx = 0;
            for (int i = t; i < nblk; i += 64) {
                const int blk = aux.y >= 0 ? aux.y + i : a.p.node_blocks[T.blk_off + blk_first + i];
                mx = max(mx, (uint32_t)vrow[blk] & 0xffffu);
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if (lane == 0) vred[warp - 10] = mx;
            asm volatile("bar.sync 3, 64;" ::: "memory");
            mx = min(max(vred[0], vred[1]), 0x7f7fu);  // inf / nan -> max finite
            const int E = (int)(mx >> 7) - 127;        // floor(log2 max |V|)
            const int s = (mx != 0 && (E >= 15 || E < -4)) ? max(E - 14, -100) : 0;
            if (t == 0) vexp[0] = s;
            const bool unit = s == 0;
            const float sc = __uint_as_float((uint32_t)(127 - s) << 23);  // 2^-s, exact
            const float2 scv = make_float2(sc, sc);
            for (int n = 0; n < NT; ++n) {
                const int st = n % SV;
                ptx::mbar_wait(&bar[V_FULL + st], (n / SV) & 1);
                if (t == 0) K1_TRACE(4, n);
                uint4 *vs = reinterpret_cast<uint4 *>(sm + C::OFF_V + st * C::KV_BYTES);
                if (unit) {
#pragma unroll 4
                    for (int c = t; c < C::KV_BYTES / 16; c += 64) {
                        uint4 w = vs[c];
                        w.x = cvt_v2(w.x, scv, true);
                        w.y = cvt_v2(w.y, scv, true);
                        w.z = cvt_v2(w.z, scv, true);
                        w.w = cvt_v2(w.w, scv, true);
                        vs[c] = w;
                    }
                } else {
#pragma unroll 4
                    for (int c = t; c < C::KV_BYTES / 16; c += 64) {
                        uint4 w = vs[c];
                        w.x = cvt_v2(w.x, scv, false);
                        w.y = cvt_v2(w.y, scv, false);
                        w.z = cvt_v2(w.z, scv, false);
                        w.w = cvt_v2(w.w, scv, false);
                        vs[c] = w;
                    }
                }
                ptx::fence_proxy_async_smem();
                if (t == 0) K1_TRACE(5, n);
                ptx::mbar_arrive(&bar[V_CONV + st]);
            }
        }
    } else {
        HALO_REGS_INC();
        // ===================== softmax warpgroups: A = warps 0-3, B = warps 4-7 =====================
        const int x = warp >> 2;                // sub-tile
        if (x == 1 && !hasB) goto done;
        {
        const int wq = warp & 3;
        const int r = wq * 32 + lane;           // sub-tile row == TMEM lane
        const int trow = x * kSubRows + r;      // tile row
        const uint32_t lane_addr = tmem + ((uint32_t)(32 * wq) << 16);
        const bool valid_row = trow < T.nrows;
        // causal prefill tile (tile_aux.z): this row (a prompt token) sees its request's first
        // aux.w + trow/g + 1 suffix tokens; every other tile sees its whole token range
        const int vis = aux.z > 0 ? aux.w + trow / a.g + 1 : 0x7fffffff;
        const int g = a.g;
        const int req = !valid_row ? 0 : aux.x >= 0 ? aux.x + trow / g : a.p.req_order[T.req_off + trow / g];
        const int head = T.kv_head * g + trow % g;
        // Q row -> smem, K-major SW128 (16-B chunk c of row r lands at chunk c ^ (r & 7)).
        // q and the partials (read by the previous layer's K2) belong to earlier kernels.
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (threadIdx.x == 0) K1_TRACE(9, 5);  // softmax: previous grid complete, q load starts
        if (!tma_q) {
            const uint4 *src = reinterpret_cast<const uint4 *>(a.q + ((int64_t)req * a.hq + head) * D);
            uint8_t *qs = sm + C::OFF_Q + x * C::Q_BYTES;
#pragma unroll
            for (int c = 0; c < D / 8; ++c) {
                const uint4 v = valid_row ? src[c] : make_uint4(0, 0, 0, 0);
                const int at = c / 8, cc = c % 8;
                *reinterpret_cast<uint4 *>(qs + at * C::ATOM_BYTES + r * 128 + ((cc ^ (r & 7)) * 16)) = v;
            }
            ptx::fence_proxy_async_smem();
            if (threadIdx.x == 0) K1_TRACE(9, 2);
            ptx::mbar_arrive(&bar[Q_FULL + x]);
        }
        const uint32_t s_addr = lane_addr + C::tmem_s(x);
        const uint32_t o_addr = lane_addr + C::tmem_o(x);
        const float c2 = a.qscale;
        const int32_t *vexp = reinterpret_cast<const int32_t *>(sm + C::OFF_VEXP);
        float m_ref = -INFINITY, l = 0.f;
        int s_cur = 0;  // the tile's V scale exponent: O accumulates P.(V 2^-s)
        for (int n = 0; n < NT; ++n) {
            ptx::mbar_wait(&bar[S_FULL + x], n & 1);
            // PV_x(n-1) has completed (S_FULL(n) commits after it, in issue order): observe its
            // phase so every PV_DONE phase is waited on (free; keeps synccheck exact)
            if (n >= 1) ptx::mbar_wait(&bar[PV_DONE + x], (n - 1) & 1);
            if (threadIdx.x == 0) K1_TRACE(6, n);
            if (threadIdx.x == 128) K1_TRACE(14, n);
            ptx::tc_fence_after();
            const int valid = min(min(kK1Tok, T.tok_end - (T.tok_begin + n * kK1Tok)),
                                  vis - (T.tok_begin + n * kK1Tok));
            // the whole 128-column score row in registers: one TMEM round trip per n-tile
            uint32_t sr[kK1Tok];
            HALO_TMEM_LD32(s_addr, sr);
            HALO_TMEM_LD32(s_addr + 32, (sr + 32));
            HALO_TMEM_LD32(s_addr + 64, (sr + 64));
            HALO_TMEM_LD32(s_addr + 96, (sr + 96));
            HALO_TMEM_WAIT_LD_REGS32(sr);
            HALO_TMEM_WAIT_LD_REGS32((sr + 32));
            HALO_TMEM_WAIT_LD_REGS32((sr + 64));
            HALO_TMEM_WAIT_LD_REGS32((sr + 96));
            if (threadIdx.x == 0) K1_TRACE_DEP(16, n, __uint_as_float(sr[0]));
            if (valid < kK1Tok) {  // only in a node's last n-tile: columns past the end -> -inf
#pragma unroll
                for (int i = 0; i < kK1Tok; ++i)
                    if (i >= valid) sr[i] = __float_as_uint(-INFINITY);
            }
            float mxv[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int i = 0; i < kK1Tok; i += 2)  // 3-input max (FMNMX3): one instruction per pair
                asm("max.f32 %0, %0, %1, %2;" : "+f"(mxv[(i >> 1) & 3]) : "f"(__uint_as_float(sr[i])), "f"(__uint_as_float(sr[i + 1])));
            const float mx = fmaxf(fmaxf(mxv[0], mxv[1]), fmaxf(mxv[2], mxv[3]));
            if (threadIdx.x == 0) K1_TRACE_DEP(10, n, mx);
            // lazy reference max: move it (and rescale O) only when a row's max grew by > 2^8
            const bool grow = mx * c2 > m_ref + kRescaleThreshold;
            if (__any_sync(0xffffffffu, grow)) {
                const float m_new = grow ? mx * c2 : m_ref;
                const float alpha = ptx::ex2(m_ref - m_new);  // 0 on a row's first tile
                if (n >= 1) {
                    ptx::mbar_wait(&bar[PV_DONE + x], (n - 1) & 1);  // O stable
                    ptx::tc_fence_after();
#pragma unroll 1
                    for (int k = 0; k < D / 32; ++k) {
                        uint32_t ov[32];
                        HALO_TMEM_LD32(o_addr + 32 * k, ov);
                        HALO_TMEM_WAIT_LD_REGS32(ov);
#pragma unroll
                        for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
                        HALO_TMEM_ST32(o_addr + 32 * k, ov);
                    }
                }
                l *= alpha;
                m_ref = m_new;
            }
            // p = 2^(s*c - m_ref) -> fp16 pairs over the consumed S columns.  Optional MUFU
            // ping-pong (HALO_K1_PINGPONG=1): A's exp pass of tile n follows B's of tile n-1 and
            // B's follows A's of tile n; measured slower than letting the two overlap (default)
            if (hasB && HALO_K1_PINGPONG) {
                // per SMSP: warp w of A pairs with warp w + 4 of B (same scheduler, same MUFU)
                if (x == 1) ptx::mbar_wait(&bar[EXP_DONE + wq], n & 1);
                else if (n >= 1) ptx::mbar_wait(&bar[EXP_DONE + 4 + wq], (n - 1) & 1);
            }
            if (threadIdx.x == 0) K1_TRACE(7, n);
            const float2 c2v = make_float2(c2, c2), nm = make_float2(-m_ref, -m_ref);
            float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                             make_float2(0.f, 0.f)};
#pragma unroll
            for (int k = 0; k < kK1Tok / 32; ++k) {
                // 32 independent exponentials back to back (one MUFU warp instruction per 8
                // cycles), four accumulators, pack, then P chunk k -> columns [16k, 16k+16)
                float2 e[16];
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    e[i] = ptx::ffma2(make_float2(__uint_as_float(sr[32 * k + 2 * i]), __uint_as_float(sr[32 * k + 2 * i + 1])), c2v, nm);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    e[i].x = ptx::ex2(e[i].x);
                    e[i].y = ptx::ex2(e[i].y);
                }
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    acc[i & 3] = ptx::fadd2(acc[i & 3], e[i]);
                    pk[i] = ptx::f2_to_h2(e[i].x, e[i].y);
                }
                HALO_TMEM_ST16(s_addr + 16 * k, pk);
            }
            const float2 a01 = ptx::fadd2(acc[0], acc[1]), a23 = ptx::fadd2(acc[2], acc[3]);
            l += (a01.x + a01.y) + (a23.x + a23.y);
            if (hasB && HALO_K1_PINGPONG) ptx::mbar_arrive(&bar[EXP_DONE + 4 * x + wq]);
            if (threadIdx.x == 0) K1_TRACE_DEP(11, n, l);
            if (threadIdx.x == 128) K1_TRACE_DEP(13, n, l);
            if (n == 0) {  // the tile's V scale (set by the converters before their first arrive)
                ptx::mbar_wait(&bar[V_CONV], 0);
                s_cur = vexp[0];
            }
            ptx::tmem_wait_st();
            if (threadIdx.x == 0) K1_TRACE(8, n);
            ptx::tc_fence_before();
            ptx::mbar_arrive(&bar[P_FULL + x]);
        }
        // ---- epilogue: O / l -> normalised partial, lse ----
        ptx::mbar_wait(&bar[PV_DONE + x], (NT - 1) & 1);
        ptx::tc_fence_after();
        const float inv = (1.f / l) * __uint_as_float((uint32_t)(127 + s_cur) << 23);  // x 2^s: exact
        // staging: sub-tile A in the K ring, B in the V ring (both idle once PV_x(NT-1) is done);
        // row r's 16-B chunks XOR-swizzled by row
        uint8_t *stage = sm + (x == 0 ? C::OFF_K : C::OFF_V);
#pragma unroll
        for (int k = 0; k < D / 32; ++k) {
            uint32_t ov[32];
            HALO_TMEM_LD32(o_addr + 32 * k, ov);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int c = k * 8 + i;
                *reinterpret_cast<float4 *>(stage + r * C::O_STRIDE + ((c ^ (r & 7)) * 16)) =
                    make_float4(__uint_as_float(ov[4 * i]) * inv, __uint_as_float(ov[4 * i + 1]) * inv,
                                __uint_as_float(ov[4 * i + 2]) * inv, __uint_as_float(ov[4 * i + 3]) * inv);
            }
        }
        const int64_t row = ((int64_t)T.slot * a.p.nreq + req) * a.hq + head;
        int64_t *row_off = reinterpret_cast<int64_t *>(sm + C::OFF_Q + x * C::Q_BYTES);  // Q_x is dead
        row_off[r] = valid_row ? row * D : -1;
        if (x == 0) asm volatile("bar.sync 1, 128;" ::: "memory");
        else asm volatile("bar.sync 2, 128;" ::: "memory");
        // each warp writes whole rows: lane = 16-B chunk (d=128: 32 chunks = 512 B per row)
        constexpr int CPR = D / 4;
        constexpr int RPI = 32 / CPR;  // rows per warp instruction
        for (int rr = wq * RPI; rr < kSubRows; rr += 4 * RPI) {
            const int row_i = rr + lane / CPR, c = lane % CPR;
            const int64_t off = row_off[row_i];
            if (off >= 0)
                reinterpret_cast<float4 *>(a.p.part_o + off)[c] =
                    *reinterpret_cast<const float4 *>(stage + row_i * C::O_STRIDE + ((c ^ (row_i & 7)) * 16));
        }
        if (valid_row) a.p.part_lse[row] = (m_ref + __log2f(l)) * kLn2;
        if (threadIdx.x == 0) K1_TRACE(9, 1);
        ptx::tc_fence_before();
        }
    }
done:
    __syncthreads();
    // completion hint for K2 (PlanDev::k1_done): this tile's partials are written (the barrier
    // orders every thread's stores before thread 0's release)
    if (threadIdx.x == 0)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.p.k1_done + (a.layer & 3)) : "memory");
    if (warp == 9) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

template <int D>
cudaError_t launch_t(const CUtensorMap *tmk, const CUtensorMap *tmv, const CUtensorMap *tmk8,
                     const CUtensorMap *tmv8, const CUtensorMap *tmq, const PrefixArgs &a, cudaStream_t s) {
    auto kern = prefix_attn_kernel<D>;
    int dev = 0;
    cudaGetDevice(&dev);
    static bool configured[64] = {};
    if (dev < 64 && !configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L1<D>::SMEM);
        if (e != cudaSuccess) return e;
        configured[dev] = true;
    }
    // programmatic dependent launch: barrier init, TMEM allocation and the tile's block list
    // overlap the previous kernel's tail (griddepcontrol.wait before any dependent access)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.p.ntiles);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = L1<D>::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, *tmk, *tmv, *tmk8, *tmv8, *tmq, a);
}

}  // namespace

cudaError_t launch_prefix_attn(const CUtensorMap *tmap_k, const CUtensorMap *tmap_v,
                               const CUtensorMap *tmap_k8, const CUtensorMap *tmap_v8,
                               const CUtensorMap *tmap_q, const PlanDev &p, const PoolGeom &g,
                               int layer, const void *q, float scale, cudaStream_t s) {
    if (p.ntiles == 0) return cudaSuccess;
    PrefixArgs a;
    a.p = p;
    a.q = static_cast<const uint16_t *>(q);
    a.hq = g.hq;
    a.hkv = g.hkv;
    a.g = g.hq / g.hkv;
    a.layer_blk = (int64_t)layer * g.cap;
    a.qscale = scale * kLog2e;
    a.tma_q = tmap_q != nullptr ? 1 : 0;
    a.vmax = g.vmax;
    a.cap = g.cap;
    a.layer = layer;
    const CUtensorMap *tq = tmap_q != nullptr ? tmap_q : tmap_k;  // unused when tma_q == 0
    if (g.d == 128) return launch_t<128>(tmap_k, tmap_v, tmap_k8, tmap_v8, tq, a, s);
    if (g.d == 64) return launch_t<64>(tmap_k, tmap_v, tmap_k8, tmap_v8, tq, a, s);
    return cudaErrorInvalidValue;
}

}  // namespace halo
