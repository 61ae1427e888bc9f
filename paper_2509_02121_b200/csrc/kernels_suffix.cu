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
//  * static schedule: the (request, kv head) units' blocks form one sequence, cut by the
//    planner into equal contiguous chunks, one per warp (148 SMs x 12 or 7 warps).  A unit cut
//    by chunk boundaries leaves one partial softmax state per piece; the last piece to
//    finish (atomic arrival counter) merges them in a fixed order -> bit-deterministic.
//  * warp-level streaming: every warp owns a ring of 2 (or 4) smem stages; its lane 0
//    issues one 1-D bulk async copy (cp.async.bulk, TMA engine) per 4-KiB K slab and V
//    slab of a 16-token block, completion on a per-stage mbarrier.  The unit's g query
//    rows (contiguous, g*d*2 bytes) arrive the same way, double-buffered, so neither a
//    block nor a unit start waits on a dependent global load.  The per-block descriptors
//    (slab index, token count, query row) are read 32 at a time with one coalesced load
//    and handed out with shuffles; the next batch is prefetched.
//  * compute from smem on CUDA cores, LPT = max(2, g, g*d/64) lanes per token row so a
//    lane holds g*d/LPT <= 64 query values and as many accumulators: each lane reads its
//    16-B chunks of a row (quarter-warp phases are 128 contiguous bytes: conflict-free),
//    fp32x2 FMAs (FFMA2) for q.k and P.V, and the g partial dot products of a row are
//    combined with a transpose-reduce (log2(LPT) + g - 1 shuffles instead of g*log2(LPT)).
//  * online softmax in base 2 with a lazy running max: o and l are rescaled only when a
//    head's block maximum exceeds the running max by more than 2^8 (exact: the final
//    state is consistent for any choice of reference max), so the common path has no
//    cross-token shuffle; l is kept per lane and reduced once per unit.
//  * K3 epilogue: merge the suffix state with the normalised fp32 K1 partials of the
//    request (slots in a fixed order), write fp32 out and lse.
#include "halo_internal.h"
#include "ptx.h"

#ifdef HALO_K2_TRACE
// Debug timeline: g_k2_trace[gw * 4 + e] = %globaltimer (ns) of global warp gw at event e:
// 0 entry, 1 first K/V stage landed, 2 K1 complete (griddepcontrol.wait returned), 3 exit.
__device__ unsigned long long *g_k2_trace = nullptr;
#define K2_TRACE(gw, ev)                                                                \
    do {                                                                                \
        if (g_k2_trace && lane == 0) {                                                  \
            unsigned long long t_;                                                      \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                    \
            g_k2_trace[(gw) * 4 + (ev)] = t_;                                           \
        }                                                                               \
    } while (0)
extern "C" int halo_debug_k2_trace(void *buf) {
    return (int)cudaMemcpyToSymbol(g_k2_trace, &buf, sizeof(buf));
}
#else
#define K2_TRACE(gw, ev) do { } while (0)
#endif

namespace halo {
namespace {

#ifndef HALO_K2_QK_BF16
#define HALO_K2_QK_BF16 0  // 1: q.k with mixed-precision bf16 FMAs (no K conversion, q kept as bf16)
#endif

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kLazy = 8.f;  // base-2 headroom of the lazy running max (p <= 2^8)

struct SuffixArgs {
    PlanDev p;
    const uint16_t *pool_k, *pool_v;  // bf16 bits
    int64_t layer_off;                // elements to this layer in the pool
    const uint16_t *q;                // [nreq][hq][D]
    float *out, *lse;
    int32_t hkv, hq;
    float qscale;                     // scale * log2(e)
};

constexpr int cmax(int a, int b) { return a > b ? a : b; }

template <int D, int G, int kWarps, int kStages>
struct Shape {
    static constexpr int LPT = cmax(2, cmax(G, G * D / 64));  // lanes per token row
    static constexpr int TPI = 32 / LPT;                      // tokens per warp iteration
    static constexpr int NIT = kBlockTok / TPI;
    static constexpr int NCH = D / (8 * LPT);                 // 16-B chunks per lane per row (q.k)
    static constexpr int SLAB = kBlockTok * D * 2;            // bytes of one (block, head) slab
    static constexpr int STAGE = 2 * SLAB;                    // K + V
    static constexpr int QB = G * D * 2;                      // the unit's q rows (bf16)
    // ring stages / q buffers: kStages and 2 unless the warps' rings would not fit in 227 KB
    static constexpr bool fits(int st, int qn) {
        return kWarps * (st * STAGE + qn * QB + kBlockTok * G * 4 + 256) <= 227 * 1024;
    }
    static constexpr int ST = fits(kStages, 1) ? kStages : kStages - 1;
    static constexpr int QN = fits(ST, 2) ? 2 : 1;
    static constexpr int OFF_Q = ST * STAGE;
    static constexpr int OFF_PS = OFF_Q + QN * QB;
    static constexpr int OFF_ALPH = OFF_PS + kBlockTok * G * 4;
    static constexpr int OFF_NT = OFF_ALPH + 8 * 4;
    static constexpr int OFF_BAR = (OFF_NT + ST * 4 + 7) / 8 * 8;
    static constexpr int WARP_SMEM = OFF_BAR + (ST + 2) * 8;
    static constexpr int WARP_SMEM_AL = (WARP_SMEM + 127) / 128 * 128;
    static_assert(G <= LPT && LPT <= 16 && NCH >= 1 && NIT >= 1, "lane mapping");
    static_assert(ST >= 2 && kWarps * WARP_SMEM_AL <= 227 * 1024, "K2 shared memory");
    static_assert(NCH * 8 * LPT == D, "d must split into 16-B chunks over the row lanes");
};

// Sum each of v[0..G) over the LPT lanes of a token group; afterwards lane c holds the
// full sum of head c / (LPT/G) in v[0].  Every lane of a head computes the same pairwise
// sums, so the replicas are bit-identical.
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

template <int D, int G>
using QAcc = float2[G][Shape<D, G, 1, 2>::NCH][4];  // q.k mapping: G heads x this lane's row chunks
template <int D, int G>
using OAcc = float2[G][D / 64];               // P.V mapping: G heads x this lane's D/32 dims

// DPL = D/32 consecutive floats at p (16-B or 8-B aligned) <-> float2 pairs
template <int NP>
__device__ __forceinline__ void ld_pairs(const float *p, float2 (&x)[NP]) {
    if constexpr (NP == 2) {
        const float4 v = *reinterpret_cast<const float4 *>(p);
        x[0] = make_float2(v.x, v.y);
        x[1] = make_float2(v.z, v.w);
    } else {
        x[0] = *reinterpret_cast<const float2 *>(p);
    }
}
template <int NP>
__device__ __forceinline__ void ld_pairs_cg(const float *p, float2 (&x)[NP]) {
    if constexpr (NP == 2) {
        const float4 v = __ldcg(reinterpret_cast<const float4 *>(p));
        x[0] = make_float2(v.x, v.y);
        x[1] = make_float2(v.z, v.w);
    } else {
        x[0] = __ldcg(reinterpret_cast<const float2 *>(p));
    }
}
template <int NP>
__device__ __forceinline__ void st_pairs(float *p, const float2 (&x)[NP], float sc) {
    if constexpr (NP == 2) {
        *reinterpret_cast<float4 *>(p) = make_float4(x[0].x * sc, x[0].y * sc, x[1].x * sc, x[1].y * sc);
    } else {
        *reinterpret_cast<float2 *>(p) = make_float2(x[0].x * sc, x[0].y * sc);
    }
}

// Final merge of a unit's suffix state (base-2 max mh, sum lh, unnormalised o) with the
// request's K1 partials, then the fp32 output / lse store.  All lanes: lane owns dims
// [lane*D/32, (lane+1)*D/32) of the G heads.
template <int D, int G>
__device__ __forceinline__ void finalize(const SuffixArgs &a, int req, int head, int nslots, int lane,
                                         const float (&mh)[G], const float (&lh)[G], OAcc<D, G> &o2,
                                         const float (&lse0)[G], bool have0) {
    constexpr int NP = D / 64, DPL = D / 32;
    const PlanDev &P = a.p;
    float M[G], L[G];
#pragma unroll
    for (int h = 0; h < G; ++h) M[h] = (lh[h] > 0.f) ? mh[h] + __log2f(lh[h]) : -INFINITY;
    const int64_t slot_stride = (int64_t)P.nreq * a.hq;
    const int64_t row0 = (int64_t)req * a.hq + head * G;
    for (int sl = 0; sl < nslots; ++sl) {
#pragma unroll
        for (int h = 0; h < G; ++h)
            M[h] = fmaxf(M[h], (sl == 0 && have0 ? lse0[h] : P.part_lse[sl * slot_stride + row0 + h]) * kLog2e);
    }
#pragma unroll
    for (int h = 0; h < G; ++h) {
        const float ws = (lh[h] > 0.f) ? ptx::ex2(mh[h] - M[h]) : 0.f;
        L[h] = lh[h] * ws;
#pragma unroll
        for (int i = 0; i < NP; ++i) o2[h][i] = ptx::fmul2(o2[h][i], make_float2(ws, ws));
    }
    for (int sl = 0; sl < nslots; ++sl) {
#pragma unroll
        for (int h = 0; h < G; ++h) {
            const int64_t row = sl * slot_stride + row0 + h;
            const float w = ptx::ex2((sl == 0 && have0 ? lse0[h] : P.part_lse[row]) * kLog2e - M[h]);
            L[h] += w;
            float2 x[NP];
            ld_pairs<NP>(P.part_o + row * D + lane * DPL, x);
#pragma unroll
            for (int i = 0; i < NP; ++i) o2[h][i] = ptx::ffma2(make_float2(w, w), x[i], o2[h][i]);
        }
    }
#pragma unroll
    for (int h = 0; h < G; ++h) {
        st_pairs<NP>(a.out + (row0 + h) * D + lane * DPL, o2[h], 1.f / L[h]);
        if (a.lse != nullptr && lane == h) a.lse[row0 + h] = (M[h] + __log2f(L[h])) * kLn2;
    }
}

template <int D, int G, int kWarps, int kStages>
__global__ void __launch_bounds__(kWarps * 32, 1) suffix_decode_kernel(const SuffixArgs a) {
    using S = Shape<D, G, kWarps, kStages>;
    constexpr int LPT = S::LPT, TPI = S::TPI, NIT = S::NIT, NCH = S::NCH, ST = S::ST;
    constexpr int NP = D / 64, DPL = D / 32;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t *ws = smem_raw + warp * S::WARP_SMEM_AL;
    uint8_t *qbuf = ws + S::OFF_Q;
    float *ps = reinterpret_cast<float *>(ws + S::OFF_PS);
    float *alph = reinterpret_cast<float *>(ws + S::OFF_ALPH);
    int32_t *snt = reinterpret_cast<int32_t *>(ws + S::OFF_NT);
    uint64_t *full = reinterpret_cast<uint64_t *>(ws + S::OFF_BAR);
    uint64_t *qbar = full + ST;

    if (lane == 0) {
        for (int s = 0; s < ST; ++s) ptx::mbar_init(&full[s], 1);
        ptx::mbar_init(&qbar[0], 1);
        ptx::mbar_init(&qbar[1], 1);
        ptx::fence_barrier_init();
    }
    __syncwarp();

    const PlanDev &P = a.p;
    const int tg = lane / LPT;   // token group within the warp
    const int c = lane % LPT;    // lane within the row
    const int hsel = c / (LPT / G);
    const bool head_writer = (c % (LPT / G)) == 0;
    const int gw = blockIdx.x * kWarps + warp;
    if (gw >= P.nwarps) return;
    K2_TRACE(gw, 0);
    const uint16_t *pk = a.pool_k + a.layer_off;
    const uint16_t *pv = a.pool_v + a.layer_off;

    // ---- producer (all lanes track the state; lane 0 issues the copies) ----
    // PDL: the next kernel in the stream (the next layer's K1) may start its prologue now;
    // it waits (griddepcontrol.wait) for this grid before touching anything K2 reads.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    int pch = gw, px = 0, phi = 0, pstart = 0;
    int4 ci = make_int4(0, 0, 0, 0);
    if (pch < P.nchunks) {
        ci = P.chunk_info[pch];
        px = pstart = ci.x;
        phi = ci.y;
    }
    uint32_t p_count = 0, c_count = 0, q_issued = 0, q_read = 0;
    int eb = -64;                       // base index of the descriptor batch in `ent`
    uint2 ent = make_uint2(0, 0), ent_next = make_uint2(0, 0);
    auto load_ent = [&](int base) {
        return (base + lane < P.nblocks) ? P.k2_ent[base + lane] : make_uint2(0, 0);
    };
    auto fill = [&]() {
        while (p_count - c_count < (uint32_t)ST) {
            if (px >= phi) {  // this warp's next chunk (only with more chunks than warps)
                if (pch >= P.nchunks) break;
                pch += P.nwarps;
                if (pch >= P.nchunks) break;
                const int4 c2 = P.chunk_info[pch];
                px = pstart = c2.x;
                phi = c2.y;
                continue;
            }
            if (px - eb >= 32 || px < eb) {
                if (px == eb + 32) {
                    ent = ent_next;
                } else {
                    ent = load_ent(px);
                }
                eb = px;
                ent_next = load_ent(eb + 32);
            }
            const int j = px - eb;
            const uint32_t ex = __shfl_sync(0xffffffffu, ent.x, j);
            const uint32_t ey = __shfl_sync(0xffffffffu, ent.y, j);
            if ((ex >> 31) || px == pstart) {  // first block of a unit in this chunk: its q rows
                if (q_issued - q_read >= (uint32_t)S::QN) break;  // q buffers busy
                if (lane == 0) {
                    const int qi = (int)(q_issued % S::QN);
                    ptx::mbar_arrive_expect_tx(&qbar[qi], S::QB);
                    ptx::bulk_g2s(qbuf + qi * S::QB, a.q + (int64_t)(ey & 0x7fffffffu) * (G * D), S::QB, &qbar[qi]);
                }
                ++q_issued;
            }
            const int st = p_count % ST;
            if (lane == 0) {
                snt[st] = (int)((ex >> kBlkCountShift) & 15u) + 1;
                const int64_t off = (int64_t)(ex & kBlkMask) * (kBlockTok * D);
                uint8_t *dst = ws + st * S::STAGE;
                ptx::mbar_arrive_expect_tx(&full[st], S::STAGE);
#ifndef HALO_K2_NO_L2_HINT
                // suffix K/V is read exactly once: an L2 evict_first policy keeps K1's
                // partials, q and the plan resident in L2 (C1 3.75 -> 4.02 M queries/s).
                // Blocks of folded prefix nodes (bit 31 of the entry) are read by several
                // units and keep the default policy.
                if (ey >> 31) {
                    ptx::bulk_g2s(dst, pk + off, S::SLAB, &full[st]);
                    ptx::bulk_g2s(dst + S::SLAB, pv + off, S::SLAB, &full[st]);
                } else {
                    const uint64_t pol = ptx::l2_policy_evict_first();
                    ptx::bulk_g2s_hint(dst, pk + off, S::SLAB, &full[st], pol);
                    ptx::bulk_g2s_hint(dst + S::SLAB, pv + off, S::SLAB, &full[st], pol);
                }
#else
                ptx::bulk_g2s(dst, pk + off, S::SLAB, &full[st]);
                ptx::bulk_g2s(dst + S::SLAB, pv + off, S::SLAB, &full[st]);
#endif
            }
            ++px;
            ++p_count;
        }
    };
    fill();

    // K1's partials (this layer's prefix attention) are read only in the epilogue and this
    // grid writes nothing before it: the streaming of the first unit piece may overlap K1
    // under programmatic dependent launch (griddepcontrol.wait before the first write).
    bool k1_ready = false;
    auto wait_k1 = [&]() {
        if (!k1_ready) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            K2_TRACE(gw, 2);
            k1_ready = true;
        }
    };
    for (int cc = gw; cc < P.nchunks; cc += P.nwarps) {
        const int4 cinfo = cc == gw ? ci : P.chunk_info[cc];
        const int lo = cinfo.x, hi = cinfo.y;
        const int u_begin = cinfo.z, u_end = cinfo.w;
        for (int u = u_begin; u < u_end; ++u) {
            const int4 m0 = P.unit_meta[2 * u], m1 = P.unit_meta[2 * u + 1];
            const int xs = max(m0.x, lo), xe = min(m0.y, hi);
            const int req = m0.z, head = m0.w;
            // once K1 is known complete, the merge's first partial lse is loaded now and
            // lands while the unit streams (the merge otherwise waits one L2 round trip)
            float lse0[G];
            const bool have0 = k1_ready && m1.x > 0 && m1.y == 1;
            if (have0) {
                const float *src = P.part_lse + (int64_t)req * a.hq + head * G;
#pragma unroll
                for (int h = 0; h < G; ++h) lse0[h] = __ldcg(src + h);
            } else {
#pragma unroll
                for (int h = 0; h < G; ++h) lse0[h] = 0.f;
            }
            OAcc<D, G> o2;
#pragma unroll
            for (int h = 0; h < G; ++h)
#pragma unroll
                for (int i = 0; i < NP; ++i) o2[h][i] = make_float2(0.f, 0.f);
            float m = -INFINITY, l = 0.f;
            if (xs < xe) {
                // q rows of the g heads, this lane's dims, pre-scaled (waits for the bulk copy)
#if HALO_K2_QK_BF16
                uint32_t qw[G][NCH][4];  // raw bf16 pairs (scale applied to the score)
#else
                QAcc<D, G> q2;           // fp32, pre-scaled
#endif
                fill();
                ptx::mbar_wait(&qbar[q_read % S::QN], (q_read / S::QN) & 1);
                const uint8_t *qs = qbuf + (q_read % S::QN) * S::QB;
#pragma unroll
                for (int h = 0; h < G; ++h)
#pragma unroll
                    for (int k = 0; k < NCH; ++k) {
                        const uint4 raw = *reinterpret_cast<const uint4 *>(qs + h * D * 2 + (k * LPT + c) * 16);
                        const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
#if HALO_K2_QK_BF16
                            qw[h][k][i] = w[i];
#else
                            const float2 f = ptx::bf2_to_f2(w[i]);
                            q2[h][k][i] = make_float2(f.x * a.qscale, f.y * a.qscale);
#endif
                        }
                    }
                __syncwarp();
                ++q_read;

                for (int x = xs; x < xe; ++x) {
                    fill();
                    const int st = c_count % ST;
                    ptx::mbar_wait(&full[st], (c_count / ST) & 1);
#ifdef HALO_K2_TRACE
                    if (c_count == 0) K2_TRACE(gw, 1);
#endif
                    const int ntok = snt[st];
                    const uint8_t *kb = ws + st * S::STAGE;
                    const uint8_t *vb = kb + S::SLAB;

                    // ---- scores: lane (tg, c) ends with head hsel's score of token it*TPI+tg
                    float s[NIT];
#pragma unroll
                    for (int it = 0; it < NIT; ++it) {
                        const int t = it * TPI + tg;
                        float2 acc[G];
#pragma unroll
                        for (int h = 0; h < G; ++h) acc[h] = make_float2(0.f, 0.f);
#pragma unroll
                        for (int k = 0; k < NCH; ++k) {
                            const uint4 raw = *reinterpret_cast<const uint4 *>(kb + t * (D * 2) + (k * LPT + c) * 16);
#if HALO_K2_QK_BF16
                            const uint32_t kw[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
                            for (int h = 0; h < G; ++h)
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    acc[h].x = ptx::fma_bf16_lo(kw[i], qw[h][k][i], acc[h].x);
                                    acc[h].y = ptx::fma_bf16_hi(kw[i], qw[h][k][i], acc[h].y);
                                }
#else
                            const float2 k0 = ptx::bf2_to_f2(raw.x), k1 = ptx::bf2_to_f2(raw.y);
                            const float2 k2 = ptx::bf2_to_f2(raw.z), k3 = ptx::bf2_to_f2(raw.w);
#pragma unroll
                            for (int h = 0; h < G; ++h) {
                                acc[h] = (k == 0) ? ptx::fmul2(q2[h][k][0], k0) : ptx::ffma2(q2[h][k][0], k0, acc[h]);
                                acc[h] = ptx::ffma2(q2[h][k][1], k1, acc[h]);
                                acc[h] = ptx::ffma2(q2[h][k][2], k2, acc[h]);
                                acc[h] = ptx::ffma2(q2[h][k][3], k3, acc[h]);
                            }
#endif
                        }
                        float part[G];
#pragma unroll
                        for (int h = 0; h < G; ++h) part[h] = acc[h].x + acc[h].y;
#if HALO_K2_QK_BF16
                        const float sc = transpose_reduce<G, LPT>(part, c) * a.qscale;
#else
                        const float sc = transpose_reduce<G, LPT>(part, c);
#endif
                        s[it] = (t < ntok) ? sc : -INFINITY;
                    }
                    // ---- lazy online softmax (base 2) ----
                    float bm = s[0];
#pragma unroll
                    for (int it = 1; it < NIT; ++it) bm = fmaxf(bm, s[it]);
                    if (__any_sync(0xffffffffu, bm > m + kLazy)) {
#pragma unroll
                        for (int msk = LPT; msk < 32; msk <<= 1)
                            bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, msk));
                        const float mn = fmaxf(m, bm);
                        const float alpha = ptx::ex2(m - mn);
                        m = mn;
                        l *= alpha;
                        if (head_writer && tg == 0) alph[hsel] = alpha;
                        __syncwarp();
#pragma unroll
                        for (int h = 0; h < G; ++h) {
                            const float al = alph[h];
#pragma unroll
                            for (int i = 0; i < NP; ++i) o2[h][i] = ptx::fmul2(o2[h][i], make_float2(al, al));
                        }
                    }
#pragma unroll
                    for (int it = 0; it < NIT; ++it) {
                        s[it] = ptx::ex2(s[it] - m);
                        l += s[it];
                    }
                    if (head_writer) {
#pragma unroll
                        for (int it = 0; it < NIT; ++it) ps[(it * TPI + tg) * G + hsel] = s[it];
                    }
                    __syncwarp();
                    // ---- o += P.V: lane owns dims [lane*DPL, +DPL) of all G heads ----
                    auto pv_token = [&](int t) {
                        float p[G];
                        if constexpr (G % 4 == 0) {
#pragma unroll
                            for (int h4 = 0; h4 < G; h4 += 4) {
                                const float4 p4 = *reinterpret_cast<const float4 *>(ps + t * G + h4);
                                p[h4] = p4.x; p[h4 + 1] = p4.y; p[h4 + 2] = p4.z; p[h4 + 3] = p4.w;
                            }
                        } else if constexpr (G == 2) {
                            const float2 p2 = *reinterpret_cast<const float2 *>(ps + t * 2);
                            p[0] = p2.x; p[1] = p2.y;
                        } else {
                            p[0] = ps[t];
                        }
                        float2 v[NP];
                        if constexpr (NP == 2) {
                            const uint2 raw = *reinterpret_cast<const uint2 *>(vb + t * (D * 2) + lane * 8);
                            v[0] = ptx::bf2_to_f2(raw.x);
                            v[1] = ptx::bf2_to_f2(raw.y);
                        } else {
                            v[0] = ptx::bf2_to_f2(*reinterpret_cast<const uint32_t *>(vb + t * (D * 2) + lane * 4));
                        }
#pragma unroll
                        for (int h = 0; h < G; ++h)
#pragma unroll
                            for (int i = 0; i < NP; ++i) o2[h][i] = ptx::ffma2(make_float2(p[h], p[h]), v[i], o2[h][i]);
                    };
                    if (ntok == kBlockTok) {
#pragma unroll
                        for (int t = 0; t < kBlockTok; ++t) pv_token(t);
                    } else {
                        for (int t = 0; t < ntok; ++t) pv_token(t);
                    }
                    __syncwarp();
                    ++c_count;
                }
                fill();
            }

            // ---- combine l over the TPI token groups (o is already per dim) ----
#pragma unroll
            for (int msk = LPT; msk < 32; msk <<= 1) l += __shfl_xor_sync(0xffffffffu, l, msk);
            // per-head (m, l) from the lane that owns each head
            float mh[G], lh[G];
#pragma unroll
            for (int h = 0; h < G; ++h) {
                mh[h] = __shfl_sync(0xffffffffu, m, h * (LPT / G));
                lh[h] = __shfl_sync(0xffffffffu, l, h * (LPT / G));
            }
            const int nslots = m1.x, nseg = m1.y;
            // first global write of this grid: the previous kernel(s) must be complete
            wait_k1();
            if (nseg == 1) {
                finalize<D, G>(a, req, head, nslots, lane, mh, lh, o2, lse0, have0);
            } else {
                // ---- stream-K: publish this piece's state; the last piece merges them all ----
                const int slot = m1.z + (cc - m1.w);
#pragma unroll
                for (int h = 0; h < G; ++h) st_pairs<NP>(P.seg_o + ((int64_t)slot * G + h) * D + lane * DPL, o2[h], 1.f);
#pragma unroll
                for (int h = 0; h < G; ++h)
                    if (lane == h) *reinterpret_cast<float2 *>(P.seg_ml + ((int64_t)slot * G + h) * 2) = make_float2(mh[h], lh[h]);
                // one acq_rel arrival by lane 0: release covers the whole warp's stores
                // (ordered before it by the warp barrier), acquire makes the other pieces'
                // stores visible to the merging warp (read from L2 with ld.cg)
                __syncwarp();
                int old = 0;
                if (lane == 0)
                    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                                 : "=r"(old) : "l"(P.unit_count + u) : "memory");
                old = __shfl_sync(0xffffffffu, old, 0);
                if (old == nseg - 1) {
                    if (lane == 0) P.unit_count[u] = 0;  // ready for the next launch
                    // merge all pieces in segment order (deterministic), from L2; the first
                    // K1 partial lse is requested up front so its latency overlaps the merge
                    float lseM[G];
                    const bool haveM = nslots > 0;
                    {
                        const float *src = P.part_lse + (int64_t)req * a.hq + head * G;
#pragma unroll
                        for (int h = 0; h < G; ++h) lseM[h] = haveM ? __ldcg(src + h) : 0.f;
                    }
                    float M[G], L[G];
#pragma unroll
                    for (int h = 0; h < G; ++h) { M[h] = -INFINITY; L[h] = 0.f; }
                    const int base = m1.z;
                    for (int sg = 0; sg < nseg; ++sg)
#pragma unroll
                        for (int h = 0; h < G; ++h)
                            M[h] = fmaxf(M[h], __ldcg(P.seg_ml + ((int64_t)(base + sg) * G + h) * 2));
#pragma unroll
                    for (int h = 0; h < G; ++h)
#pragma unroll
                        for (int i = 0; i < NP; ++i) o2[h][i] = make_float2(0.f, 0.f);
                    for (int sg = 0; sg < nseg; ++sg) {
#pragma unroll
                        for (int h = 0; h < G; ++h) {
                            const float2 ml = __ldcg(reinterpret_cast<const float2 *>(
                                P.seg_ml + ((int64_t)(base + sg) * G + h) * 2));
                            const float w = (ml.y > 0.f) ? ptx::ex2(ml.x - M[h]) : 0.f;
                            L[h] += ml.y * w;
                            float2 x[NP];
                            ld_pairs_cg<NP>(P.seg_o + ((int64_t)(base + sg) * G + h) * D + lane * DPL, x);
#pragma unroll
                            for (int i = 0; i < NP; ++i) o2[h][i] = ptx::ffma2(make_float2(w, w), x[i], o2[h][i]);
                        }
                    }
                    finalize<D, G>(a, req, head, nslots, lane, M, L, o2, lseM, haveM);

                }
            }
            __syncwarp();
        }
    }
    K2_TRACE(gw, 3);
}

template <int D, int G, int kWarps, int kStages>
cudaError_t launch_t(const SuffixArgs &a, cudaStream_t s) {
    using S = Shape<D, G, kWarps, kStages>;
    const int smem = kWarps * S::WARP_SMEM_AL;
    auto kern = suffix_decode_kernel<D, G, kWarps, kStages>;
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
    // programmatic dependent launch: CTAs may start while K1 (the previous kernel) drains
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.p.ntiles > 0 ? 1 : 0;  // overlap K1 only (never a previous K2)
    return cudaLaunchKernelEx(&cfg, kern, a);
}

}  // namespace

cudaError_t launch_suffix_decode(const PlanDev &p, const PoolGeom &g, const void *pool_k,
                                 const void *pool_v, int layer, const void *q, float *out,
                                 float *lse, float scale, int num_sms, cudaStream_t s) {
    (void)num_sms;  // the grid follows the plan's warp count
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
#define HALO_K2_CASE(DD, GG)                                                                       \
    if (g.d == DD && G == GG)                                                                      \
        return p.k2_warps == kK2WarpsNarrow ? launch_t<DD, GG, kK2WarpsNarrow, kK2StagesNarrow>(a, s) \
                                            : launch_t<DD, GG, kK2WarpsWide, kK2StagesWide>(a, s);
    HALO_K2_CASE(128, 1) HALO_K2_CASE(128, 2) HALO_K2_CASE(128, 4) HALO_K2_CASE(128, 8)
    HALO_K2_CASE(64, 1) HALO_K2_CASE(64, 2) HALO_K2_CASE(64, 4) HALO_K2_CASE(64, 8)
#undef HALO_K2_CASE
    return cudaErrorInvalidValue;
}

}  // namespace halo
