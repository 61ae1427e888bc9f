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
//    by chunk boundaries leaves one partial softmax state per piece; the unit's first piece
//    (the last unit of its chunk) merges them once the others have arrived (otherwise the
//    last piece to arrive does), in a fixed order -> bit-deterministic.
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
// 0 entry, 1 first K/V stage landed, 2 K1 complete (griddepcontrol.wait returned), 3 exit,
// 4 last K/V stage landed, 5 start of the last unit end (merge / finalize / publish),
// 6 before the completion-count atomic.
__device__ unsigned long long *g_k2_trace = nullptr;
#define K2_TRACE(gw, ev)                                                                \
    do {                                                                                \
        if (g_k2_trace && lane == 0) {                                                  \
            unsigned long long t_;                                                      \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                    \
            g_k2_trace[(gw) * 8 + (ev)] = t_;                                           \
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

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kLazy = 8.f;  // base-2 headroom of the lazy running max (p <= 2^8)
constexpr int NPAD = kK2HeadPad;  // MMA N: the unit's g q-heads padded to 8
constexpr int NPARK = 16;         // units a warp may park while K1 is still running
#ifndef HALO_K2_EXP
#define HALO_K2_EXP 0             // timing experiments only: 1 = skip block compute, 2 = skip unit end
#endif
#ifndef HALO_K2_PF
#define HALO_K2_PF 0              // blocks prefetched into L2 ahead of the smem ring (A/B: 2-8 slower, tools/k1k2_cosched_sweep.py)
#endif

struct SuffixArgs {
    PlanDev p;
    int64_t layer_blk;                // layer * cap (4th TMA coordinate offset)
    const uint16_t *q;                // [nreq][hq][D]
    float *out, *lse;
    int32_t hkv, hq;
    float qscale;                     // scale * log2(e)
    int32_t layer;                    // selects the dynamic-claim counter (layer % 4)
};

template <int D, int G, int kWarps, int kStages>
struct Shape {
    static constexpr int KS = D / 16;                         // k-steps of q.k = m-tiles of P.V
    static constexpr int ATOMS = D / 64;                      // 128-B swizzle atoms per row
    static constexpr int SLAB = kBlockTok * D * 2;            // bytes of one (block, head) slab
    static constexpr int STAGE = 2 * SLAB;                    // K + V (multiple of 1024)
    static constexpr int QB = G * D * 2;                      // the unit's q rows (bf16)
    // per-warp misc area: q buffers, alpha, token counts, chunk FIFO, barriers
    static constexpr int misc(int st, int qn) { return (qn * QB + 8 * 4 + st * 4 + 8 * 4 + NPARK * 4 + (st + 2) * 8 + 127) / 128 * 128; }
    static constexpr bool fits(int st, int qn) { return st >= 1 && kWarps * (st * STAGE + misc(st, qn)) <= 227 * 1024; }
    // ring stages / q buffers: kStages and 2 unless the warps' areas would not fit in 227 KB
    static constexpr int ST = fits(kStages, 1) ? kStages : fits(kStages - 1, 1) ? kStages - 1 : kStages - 2;
    static constexpr int QN = fits(ST, 2) ? 2 : 1;
    static constexpr int MISC = misc(ST, QN);
    static constexpr int OFF_MISC = kWarps * ST * STAGE;      // stages of all warps first (1024-aligned)
    static constexpr int OFF_Q = 0;                           // within the misc area
    static constexpr int OFF_ALPH = OFF_Q + QN * QB;
    static constexpr int OFF_NT = OFF_ALPH + 8 * 4;
    static constexpr int OFF_CQ = OFF_NT + ST * 4;
    static constexpr int OFF_PARK = OFF_CQ + 8 * 4;               // [NPARK] parked units
    static constexpr int OFF_BAR = (OFF_PARK + NPARK * 4 + 7) / 8 * 8;
    static constexpr int SMEM = OFF_MISC + kWarps * MISC;
    static_assert(ST >= 2 && SMEM <= 227 * 1024, "K2 shared memory");
    static_assert(STAGE % 1024 == 0 && G <= NPAD && D % 64 == 0, "K2 shape");
};

// Byte offset of (token r, dim d) in a (block, head) slab loaded by TMA with 128-B swizzle:
// atom d/64 of 16 rows x 128 B; 16-B chunk c of row r sits at chunk c ^ (r % 8).
__device__ __forceinline__ uint32_t swz(int r, int d) {
    return (uint32_t)((d >> 6) * (kBlockTok * 128) + r * 128 + ((((d & 63) >> 3) ^ (r & 7)) << 4));
}

// Final merge of a unit's suffix state with the request's K1 partials, then the fp32 output /
// lse store.  Lane layout (the P.V MMA's accumulator): lane (g = lane/4, c = lane%4) holds, for
// heads h_e = 2c + e (e = 0, 1) and dims d = 16t + g + 8j, o[t][2j + e].  mh/lh: base-2 running
// max and the (lane-reduced) sum of the two heads.  Online over the slots (fixed order: bit-
// deterministic): a slot's lse and o rows are loaded together, one memory round trip per slot
// (round 1 loaded all lse first, then the o rows: two).
template <int D, int G>
__device__ __forceinline__ void finalize(const SuffixArgs &a, int req, int head, int nslots, int lane,
                                         const float (&mh)[2], const float (&lh)[2], float (&o)[D / 16][4]) {
    constexpr int KS = D / 16;
    const PlanDev &P = a.p;
    const int g = lane >> 2, c = lane & 3;
    const int64_t slot_stride = (int64_t)P.nreq * a.hq;
    const int64_t row0 = (int64_t)req * a.hq + head * G;
    // lanes of padding heads (2c + e >= G) read head 0's rows (valid addresses; results unused)
    const int64_t r0 = row0 + (2 * c < G ? 2 * c : 0), r1 = row0 + (2 * c + 1 < G ? 2 * c + 1 : 0);
    float xl[2], xo[KS][4];
    auto load_slot = [&](int sl) {
        const int64_t s = (int64_t)sl * slot_stride;
        xl[0] = __ldcg(P.part_lse + s + r0);
        xl[1] = __ldcg(P.part_lse + s + r1);
        const float *s0 = P.part_o + (s + r0) * D + g, *s1 = P.part_o + (s + r1) * D + g;
#pragma unroll
        for (int t = 0; t < KS; ++t) {
            xo[t][0] = __ldcg(s0 + 16 * t);
            xo[t][2] = __ldcg(s0 + 16 * t + 8);
            xo[t][1] = __ldcg(s1 + 16 * t);
            xo[t][3] = __ldcg(s1 + 16 * t + 8);
        }
    };
    float M[2], L[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        M[e] = lh[e] > 0.f ? mh[e] : -INFINITY;
        L[e] = lh[e];
    }
    for (int sl = 0; sl < nslots; ++sl) {
        load_slot(sl);  // lse and o rows of the slot: one round trip
        float cl[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) cl[e] = xl[e] * kLog2e;
        float (&co)[KS][4] = xo;
        float al[2], w[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const float mn = fmaxf(M[e], cl[e]);
            al[e] = ptx::ex2(M[e] - mn);  // 0 while M is -inf (no suffix tokens yet)
            w[e] = ptx::ex2(cl[e] - mn);
            L[e] = L[e] * al[e] + w[e];
            M[e] = mn;
        }
#pragma unroll
        for (int t = 0; t < KS; ++t) {
            o[t][0] = fmaf(w[0], co[t][0], o[t][0] * al[0]);
            o[t][2] = fmaf(w[0], co[t][2], o[t][2] * al[0]);
            o[t][1] = fmaf(w[1], co[t][1], o[t][1] * al[1]);
            o[t][3] = fmaf(w[1], co[t][3], o[t][3] * al[1]);
        }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int h = 2 * c + e;
        if (h >= G) continue;
        const float inv = 1.f / L[e];
        float *dst = a.out + (row0 + h) * D + g;
#pragma unroll
        for (int t = 0; t < KS; ++t) {
            dst[16 * t] = o[t][e] * inv;
            dst[16 * t + 8] = o[t][2 + e] * inv;
        }
        if (a.lse != nullptr && g == 0) a.lse[row0 + h] = (M[e] + __log2f(L[e])) * kLn2;
    }
}

template <int D, int G, int kWarps, int kStages>
__global__ void __launch_bounds__(kWarps * 32, 1)
suffix_decode_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                     const SuffixArgs a) {
    using S = Shape<D, G, kWarps, kStages>;
    constexpr int KS = S::KS, ST = S::ST;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t *stages = smem_raw + warp * ST * S::STAGE;
    uint8_t *ms = smem_raw + S::OFF_MISC + warp * S::MISC;
    uint8_t *qbuf = ms + S::OFF_Q;
    float *alph = reinterpret_cast<float *>(ms + S::OFF_ALPH);
    int32_t *snt = reinterpret_cast<int32_t *>(ms + S::OFF_NT);
    uint64_t *full = reinterpret_cast<uint64_t *>(ms + S::OFF_BAR);
    uint64_t *qbar = full + ST;
    (void)alph;

    if (lane == 0) {
        for (int s = 0; s < ST; ++s) ptx::mbar_init(&full[s], 1);
        for (int i = 0; i < S::QN; ++i) ptx::mbar_init(&qbar[i], 1);
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tmk);
        ptx::prefetch_tmap(&tmv);
    }
    __syncwarp();

    const PlanDev &P = a.p;
    const int g = lane >> 2, c = lane & 3;
    const int gw = blockIdx.x * kWarps + warp;
    if (gw >= P.nwarps) return;
    K2_TRACE(gw, 0);

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
    // static-then-dynamic schedule (optional, halo_plan_options.k2_tail_pct): after its static
    // chunk the warp claims chunks from a per-layer counter; the next claim is issued when a
    // chunk starts (lane 0 holds the result).  Chunk ids go through a small per-warp FIFO from
    // the producer (fill) to the consumer loop.
    const bool dyn = P.dyn_first < P.nchunks;
    const int ndyn = P.nchunks - P.dyn_first;
    int32_t *dcount = P.dyn_counter + (a.layer & 3);
    int32_t *cq = reinterpret_cast<int32_t *>(ms + S::OFF_CQ);
    uint32_t cq_w = 0, cq_r = 0;
    bool prod_done = false;
    int claim = 0;
    if (dyn) {
        if (lane == 0) {
            cq[0] = gw;
            claim = atomicAdd(dcount, 1);
        }
        cq_w = 1;
    }
    uint32_t p_count = 0, c_count = 0, q_issued = 0, q_read = 0;
    int eb = -64;                       // base index of the descriptor batch in `ent`
    uint2 ent = make_uint2(0, 0), ent_next = make_uint2(0, 0);
    auto load_ent = [&](int base) {
        return (base + lane < P.nblocks) ? P.k2_ent[base + lane] : make_uint2(0, 0);
    };
    auto fill = [&]() {
        while (p_count - c_count < (uint32_t)ST) {
            if (px >= phi) {  // this warp's next chunk
                if (!dyn) {   // static round-robin (only with more chunks than warps)
                    if (pch >= P.nchunks) break;
                    pch += P.nwarps;
                    if (pch >= P.nchunks) break;
                } else {
                    if (prod_done || cq_w - cq_r >= 8) break;
                    const int k = __shfl_sync(0xffffffffu, claim, 0);
                    if (k >= ndyn) {  // no work left; the launch's last claim resets the counter
                        prod_done = true;
                        if (lane == 0 && k == ndyn + P.nwarps - 1) atomicExch(dcount, 0);
                        break;
                    }
                    pch = P.dyn_first + k;
                    if (lane == 0) {
                        cq[cq_w & 7] = pch;
                        claim = atomicAdd(dcount, 1);  // the claim after this one, in flight
                    }
                    ++cq_w;
                }
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
                const uint32_t slab = ex & kBlkMask;
                const int blk = (int)(slab / (uint32_t)a.hkv), hd = (int)(slab % (uint32_t)a.hkv);
                const int c3 = (int)(a.layer_blk + blk);
                uint8_t *dst = stages + st * S::STAGE;
                ptx::mbar_arrive_expect_tx(&full[st], S::STAGE);
                // K and V slabs by TMA in the 128-B swizzle the ldmatrix reads expect.  Suffix
                // K/V is read exactly once: L2 evict_first keeps K1's partials, q and the plan
                // resident (C1 3.75 -> 4.02 M queries/s, round 1); blocks of folded prefix nodes
                // (bit 31 of the entry) are read by several units and keep the default policy.
                if (ey >> 31) {
#pragma unroll
                    for (int at = 0; at < S::ATOMS; ++at) {
                        ptx::tma_load_4d(dst + at * (kBlockTok * 128), &tmk, at * 64, 0, hd, c3, &full[st]);
                        ptx::tma_load_4d(dst + S::SLAB + at * (kBlockTok * 128), &tmv, at * 64, 0, hd, c3, &full[st]);
                    }
                } else {
                    const uint64_t pol = ptx::l2_policy_evict_first();
#pragma unroll
                    for (int at = 0; at < S::ATOMS; ++at) {
                        ptx::tma_load_4d_hint(dst + at * (kBlockTok * 128), &tmk, at * 64, 0, hd, c3, &full[st], pol);
                        ptx::tma_load_4d_hint(dst + S::SLAB + at * (kBlockTok * 128), &tmv, at * 64, 0, hd, c3,
                                              &full[st], pol);
                    }
                }
            }
            // L2 prefetch HALO_K2_PF blocks ahead (same chunk): the ring's smem stages cap the
            // bytes a warp has in flight; prefetched blocks raise it without holding smem, so
            // the SMs left free beside K1 can stream closer to HBM speed
            if (HALO_K2_PF > 0 && px + HALO_K2_PF < phi) {
                const int jp = px + HALO_K2_PF - eb;  // < 64: within ent / ent_next
                const uint32_t pex = jp < 32 ? __shfl_sync(0xffffffffu, ent.x, jp)
                                             : __shfl_sync(0xffffffffu, ent_next.x, jp - 32);
                if (lane == 0) {
                    const uint32_t slab = pex & kBlkMask;
                    const int blk = (int)(slab / (uint32_t)a.hkv), hd = (int)(slab % (uint32_t)a.hkv);
#pragma unroll
                    for (int at = 0; at < S::ATOMS; ++at) {
                        ptx::tma_prefetch_4d(&tmk, at * 64, 0, hd, (int)(a.layer_blk + blk));
                        ptx::tma_prefetch_4d(&tmv, at * 64, 0, hd, (int)(a.layer_blk + blk));
                    }
                }
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
    // this layer slot's scratch (a K2 launch may overlap the previous layer's)
    const int ls = a.layer & 3;
    float *seg_o = P.seg_o + ls * P.seg_slot_stride;
    float *seg_ml = P.seg_ml + ls * P.seg_slot_stride;
    int32_t *unit_count = P.unit_count + ls * P.count_slot_stride;
    constexpr int PARK_UNIT = G * (D + 2);
    float *park = P.park + (int64_t)ls * P.nunits * PARK_UNIT;
    int32_t *plist = reinterpret_cast<int32_t *>(ms + S::OFF_PARK);
    int npark = 0;
    // has K1 finished (all its CTAs published)?  A hint only: outputs are written after
    // griddepcontrol.wait either way.  Lane 0 polls the completion counter once per block with
    // a non-blocking load whose value is read one block later, so the unit ends find the
    // answer without a round trip.
    uint32_t k1_poll = 0;     // lane 0: the last poll (possibly still in flight)
    bool k1_polled = false, k1_seen = false;
    auto k1_poll_issue = [&]() {
        if (lane == 0) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(k1_poll) : "l"(P.k1_done + ls));
        k1_polled = true;
    };
    auto k1_poll_check = [&]() {
        if (!k1_ready && !k1_seen && k1_polled && __shfl_sync(0xffffffffu, k1_poll, 0) >= (uint32_t)P.ntiles)
            k1_seen = true;
    };
    auto k1_hint = [&]() -> bool {
        if (k1_ready || k1_seen) return true;
        if (k1_polled) {
            k1_poll_check();
            return k1_seen;
        }
        uint32_t v = 0;
        if (lane == 0) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(P.k1_done + ls) : "memory");
        v = __shfl_sync(0xffffffffu, v, 0);
        return v >= (uint32_t)P.ntiles;
    };
    // merge every stream-K piece of unit u (in segment order: deterministic) and finalize;
    // online over the pieces, each piece's (m, l) and o loaded together
    // `own` >= 0: this warp's piece of the unit, whose state (om, ol, oo) is still in registers
    // (not re-read from L2: one round trip less at the end of the kernel)
    auto merge_pieces = [&](int u, int own, const float (&om)[2], const float (&ol)[2], const float (&oo)[KS][4]) {
        const int4 m0 = P.unit_meta[2 * u], m1 = P.unit_meta[2 * u + 1];
        const int req = m0.z, head = m0.w, nslots = m1.x, nseg = m1.y, base = m1.z;
        const int c2 = 2 * c < G ? 2 * c : 0;  // padding-head lanes read head 0 (results unused)
        float2 xml[2];
        float4 xo[KS];
        auto load_seg = [&](int sg) {
            if (sg == own) {
#pragma unroll
                for (int e = 0; e < 2; ++e) xml[e] = make_float2(om[e], ol[e]);
#pragma unroll
                for (int t = 0; t < KS; ++t) xo[t] = make_float4(oo[t][0], oo[t][1], oo[t][2], oo[t][3]);
                return;
            }
            const int64_t sidx = base + sg;
#pragma unroll
            for (int e = 0; e < 2; ++e)
                xml[e] = __ldcg(reinterpret_cast<const float2 *>(seg_ml + (sidx * NPAD + (2 * c + e < G ? 2 * c + e : c2)) * 2));
            const float *src = seg_o + sidx * (NPAD * D) + (2 * c < G ? lane : 0) * (4 * KS);
#pragma unroll
            for (int t = 0; t < KS; ++t) xo[t] = __ldcg(reinterpret_cast<const float4 *>(src + 4 * t));
        };
        float M[2] = {-INFINITY, -INFINITY}, L[2] = {0.f, 0.f};
        float o[KS][4];
#pragma unroll
        for (int t = 0; t < KS; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
        for (int sg = 0; sg < nseg; ++sg) {
            load_seg(sg);  // the piece's (m, l) and o: one round trip
            const float2 (&cml)[2] = xml;
            const float4 (&co)[KS] = xo;
            float al[2], w[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                if (cml[e].y > 0.f) {  // a piece with tokens (l > 0): fold it in
                    const float mn = fmaxf(M[e], cml[e].x);
                    al[e] = ptx::ex2(M[e] - mn);
                    w[e] = ptx::ex2(cml[e].x - mn);
                    L[e] = L[e] * al[e] + cml[e].y * w[e];
                    M[e] = mn;
                } else {
                    al[e] = 1.f;
                    w[e] = 0.f;
                }
            }
#pragma unroll
            for (int t = 0; t < KS; ++t) {
                o[t][0] = fmaf(w[0], co[t].x, o[t][0] * al[0]);
                o[t][1] = fmaf(w[1], co[t].y, o[t][1] * al[1]);
                o[t][2] = fmaf(w[0], co[t].z, o[t][2] * al[0]);
                o[t][3] = fmaf(w[1], co[t].w, o[t][3] * al[1]);
            }
        }
        finalize<D, G>(a, req, head, nslots, lane, M, L, o);
    };
    // wait for K1, then merge the parked units (whole units from `park`, stream-K ones from
    // their pieces) in parking order
    auto drain = [&]() {
        wait_k1();
        __syncwarp();
        const float zm[2] = {0.f, 0.f}, zo[KS][4] = {};  // (parked pieces: all state in L2)
        for (int i = 0; i < npark; ++i) {
            const int ent = plist[i];
            const int u = ent & 0x7fffffff;
            if (ent < 0) {
                merge_pieces(u, -1, zm, zm, zo);
                continue;
            }
            const int4 m0 = P.unit_meta[2 * u], m1 = P.unit_meta[2 * u + 1];
            const float *pk = park + (int64_t)u * PARK_UNIT;
            float o[KS][4], mm[2] = {-INFINITY, -INFINITY}, ll[2] = {0.f, 0.f};
#pragma unroll
            for (int t = 0; t < KS; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int h = 2 * c + e;
                if (h >= G) continue;
#pragma unroll
                for (int t = 0; t < KS; ++t) {
                    o[t][e] = __ldcg(pk + h * D + 16 * t + g);
                    o[t][2 + e] = __ldcg(pk + h * D + 16 * t + g + 8);
                }
                const float2 ml = __ldcg(reinterpret_cast<const float2 *>(pk + G * D + 2 * h));
                mm[e] = ml.x;
                ll[e] = ml.y;
            }
            finalize<D, G>(a, m0.z, m0.w, m1.x, lane, mm, ll, o);
        }
        __syncwarp();
        npark = 0;
    };
    // per-lane ldmatrix row addresses within a slab: K (A operand, row = token) and V^T
    // (A operand via .trans, memory row = token); matrix m = lane / 8, row lane % 8
    const int lm = lane >> 3, lr = lane & 7;
    const int k_tok = lr + 8 * (lm & 1), k_d = 8 * (lm >> 1);   // K: a0..a3 = (tok 0-7 | 8-15) x (d +0 | +8)
    const int v_tok = lr + 8 * (lm >> 1), v_d = 8 * (lm & 1);   // V^T: a0..a3 = (d +0 | +8) x (tok 0-7 | 8-15)
    const int e_src = 8 * c + (g >> 1);  // lane holding p(token 2c, head g) (and 2c+1 at +4)
    for (uint32_t ck = 0;; ++ck) {
        int cc;
        if (!dyn) {
            cc = gw + (int)ck * P.nwarps;
            if (cc >= P.nchunks) break;
        } else {
            while (cq_w <= ck && !prod_done) fill();  // the producer decides the next chunk
            if (ck >= cq_w) break;
            __syncwarp();
            cc = cq[ck & 7];
            __syncwarp();
            cq_r = ck + 1;
        }
        const int4 cinfo = cc == gw ? ci : P.chunk_info[cc];
        const int lo = cinfo.x, hi = cinfo.y;
        const int u_begin = cinfo.z, u_end = cinfo.w;
        for (int u = u_begin; u < u_end; ++u) {
            const int4 m0 = P.unit_meta[2 * u], m1 = P.unit_meta[2 * u + 1];
            const int xs = max(m0.x, lo), xe = min(m0.y, hi);
            const int req = m0.z, head = m0.w;
            // O^T accumulators (d x 8 heads, MMA C layout), running max / lane-partial sums
            float o[KS][4];
#pragma unroll
            for (int t = 0; t < KS; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
            float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
            if (xs < xe) {
                // q^T as the B operand of q.k: b0 = q[head g][16s + 2c, +1], b1 = +8 (0 for g >= G)
                uint32_t qf[KS][2];
                fill();
                ptx::mbar_wait(&qbar[q_read % S::QN], (q_read / S::QN) & 1);
                const uint8_t *qs = qbuf + (q_read % S::QN) * S::QB;
#pragma unroll
                for (int t = 0; t < KS; ++t) {
                    qf[t][0] = g < G ? *reinterpret_cast<const uint32_t *>(qs + (g * D + 16 * t + 2 * c) * 2) : 0u;
                    qf[t][1] = g < G ? *reinterpret_cast<const uint32_t *>(qs + (g * D + 16 * t + 8 + 2 * c) * 2) : 0u;
                }
                __syncwarp();
                ++q_read;

                for (int x = xs; x < xe; ++x) {
                    fill();
                    if (!k1_ready && !k1_seen) {  // refresh the K1 completion hint
                        k1_poll_check();
                        if (!k1_seen) k1_poll_issue();
                    }
                    const int st = c_count % ST;
                    ptx::mbar_wait(&full[st], (c_count / ST) & 1);
#ifdef HALO_K2_TRACE
                    if (c_count == 0) K2_TRACE(gw, 1);
                    K2_TRACE(gw, 4);
#endif
                    if (HALO_K2_EXP & 1) { __syncwarp(); ++c_count; continue; }
                    const int ntok = snt[st];
                    const uint32_t kb = ptx::smem_u32(stages + st * S::STAGE);
                    const uint32_t vb = kb + S::SLAB;

                    // ---- S^T (16 tokens x 8 heads) = K . q^T on the tensor cores ----
                    float sc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int t = 0; t < KS; ++t) {
                        uint32_t a0, a1, a2, a3;
                        ptx::ldsm_x4(kb + swz(k_tok, 16 * t + k_d), a0, a1, a2, a3);
                        ptx::mma_16816(sc, a0, a1, a2, a3, qf[t][0], qf[t][1]);
                    }
                    // lane holds tokens g, g+8 of heads 2c, 2c+1: scale, mask padding and the
                    // tokens past a partial block
                    float s4[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int tok = g + 8 * (i >> 1), hh = 2 * c + (i & 1);
                        s4[i] = (tok < ntok && hh < G) ? sc[i] * a.qscale : -INFINITY;
                    }
                    // ---- lazy online softmax (base 2): rescale only when a head's block max
                    // exceeds its running max by more than 2^8 ----
                    const float bm0 = fmaxf(s4[0], s4[2]), bm1 = fmaxf(s4[1], s4[3]);
                    if (__any_sync(0xffffffffu, bm0 > m[0] + kLazy || bm1 > m[1] + kLazy)) {
                        float r0 = bm0, r1 = bm1;
#pragma unroll
                        for (int msk = 4; msk < 32; msk <<= 1) {
                            r0 = fmaxf(r0, __shfl_xor_sync(0xffffffffu, r0, msk));
                            r1 = fmaxf(r1, __shfl_xor_sync(0xffffffffu, r1, msk));
                        }
                        const float n0 = fmaxf(m[0], r0), n1 = fmaxf(m[1], r1);
                        const float al0 = n0 == -INFINITY ? 1.f : ptx::ex2(m[0] - n0);
                        const float al1 = n1 == -INFINITY ? 1.f : ptx::ex2(m[1] - n1);
                        m[0] = n0;
                        m[1] = n1;
                        l[0] *= al0;
                        l[1] *= al1;
#pragma unroll
                        for (int t = 0; t < KS; ++t) {
                            o[t][0] *= al0;
                            o[t][2] *= al0;
                            o[t][1] *= al1;
                            o[t][3] *= al1;
                        }
                    }
                    float p[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float mm = m[i & 1];
                        p[i] = mm == -INFINITY ? 0.f : ptx::ex2(s4[i] - mm);
                    }
                    l[0] += p[0] + p[2];
                    l[1] += p[1] + p[3];
                    // ---- P^T as the B operand of P.V: lane (g, c) needs p(token 2c, 2c+1 | +8,
                    // head g), held by lanes 8c + g/2 (+4) -> 8 shuffles, then an exact bf16
                    // hi + lo split (P carries ~16 bits into the fp32 accumulation) ----
                    const bool odd = g & 1;
                    float q0, q1, q2, q3;
                    {
                        const float x0 = __shfl_sync(0xffffffffu, p[0], e_src), x1 = __shfl_sync(0xffffffffu, p[1], e_src);
                        const float y0 = __shfl_sync(0xffffffffu, p[0], e_src + 4), y1 = __shfl_sync(0xffffffffu, p[1], e_src + 4);
                        const float z0 = __shfl_sync(0xffffffffu, p[2], e_src), z1 = __shfl_sync(0xffffffffu, p[3], e_src);
                        const float w0 = __shfl_sync(0xffffffffu, p[2], e_src + 4), w1 = __shfl_sync(0xffffffffu, p[3], e_src + 4);
                        q0 = odd ? x1 : x0;   // p(2c, g)
                        q1 = odd ? y1 : y0;   // p(2c+1, g)
                        q2 = odd ? z1 : z0;   // p(2c+8, g)
                        q3 = odd ? w1 : w0;   // p(2c+9, g)
                    }
                    const uint32_t bh0 = ptx::f2_to_bf2(q0, q1), bh1 = ptx::f2_to_bf2(q2, q3);
                    const float2 r01 = ptx::bf2_to_f2(bh0), r23 = ptx::bf2_to_f2(bh1);
                    const uint32_t bl0 = ptx::f2_to_bf2(q0 - r01.x, q1 - r01.y);
                    const uint32_t bl1 = ptx::f2_to_bf2(q2 - r23.x, q3 - r23.y);
                    // ---- O^T (d x 8 heads) += V^T . P^T ----
#pragma unroll
                    for (int t = 0; t < KS; ++t) {
                        uint32_t a0, a1, a2, a3;
                        ptx::ldsm_x4_t(vb + swz(v_tok, 16 * t + v_d), a0, a1, a2, a3);
                        ptx::mma_16816(o[t], a0, a1, a2, a3, bh0, bh1);
                        ptx::mma_16816(o[t], a0, a1, a2, a3, bl0, bl1);
                    }
                    __syncwarp();
                    ++c_count;
                }
                fill();
            }

            // ---- the unit's per-head sums over the 8 lanes of each head pair ----
#pragma unroll
            for (int msk = 4; msk < 32; msk <<= 1) {
                l[0] += __shfl_xor_sync(0xffffffffu, l[0], msk);
                l[1] += __shfl_xor_sync(0xffffffffu, l[1], msk);
            }
            const int nslots = m1.x, nseg = m1.y;
            K2_TRACE(gw, 5);
            if (HALO_K2_EXP & 2) { __syncwarp(); continue; }
            if (nseg == 1) {
                if (k1_hint()) {
                    wait_k1();  // first output write of this grid: K1 (and before it the previous K2) done
                    finalize<D, G>(a, req, head, nslots, lane, m, l, o);
                } else {
                    // K1 still runs: park the unit's state (L2) and stream on; merged by drain()
                    float *pk = park + (int64_t)u * PARK_UNIT;
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int h = 2 * c + e;
                        if (h >= G) continue;
#pragma unroll
                        for (int t = 0; t < KS; ++t) {
                            pk[h * D + 16 * t + g] = o[t][e];
                            pk[h * D + 16 * t + g + 8] = o[t][2 + e];
                        }
                        if (g == 0) *reinterpret_cast<float2 *>(pk + G * D + 2 * h) = make_float2(m[e], l[e]);
                    }
                    if (lane == 0) plist[npark] = u;
                    ++npark;
                    if (npark == NPARK) drain();
                }
            } else {
                // ---- stream-K piece ----
                // Static schedules with one chunk per warp: the unit's FIRST piece (segment 0 --
                // always the last unit of its chunk, so every other piece sits at the start or
                // middle of another warp's chunk and never waits) merges: the other pieces
                // publish and arrive without a return value, the merger waits for their count
                // with an acquire poll and folds its own state from registers (no publish, no
                // arrival round trip).  Otherwise the last piece to arrive merges.
                const int own = cc - m1.w;
                const bool designated = !dyn && P.nchunks <= P.nwarps;
                auto publish = [&]() {
                    const int slot = m1.z + own;
                    float *so = seg_o + (int64_t)slot * (NPAD * D) + lane * (4 * KS);
                    if (2 * c < G) {
#pragma unroll
                        for (int t = 0; t < KS; ++t) *reinterpret_cast<float4 *>(so + 4 * t) = make_float4(o[t][0], o[t][1], o[t][2], o[t][3]);
                    }
                    if (g == 0) {
#pragma unroll
                        for (int e = 0; e < 2; ++e)
                            if (2 * c + e < G)
                                *reinterpret_cast<float2 *>(seg_ml + ((int64_t)slot * NPAD + 2 * c + e) * 2) = make_float2(m[e], l[e]);
                    }
                    __syncwarp();  // the warp's stores before lane 0's release
                };
                if (designated && own == 0) {
                    if (lane == 0) {  // the other pieces' arrivals (release): acquire
                        uint32_t v;
                        for (;;) {
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(unit_count + u) : "memory");
                            if (v >= (uint32_t)(nseg - 1)) break;
                            __nanosleep(100);
                        }
                        unit_count[u] = 0;  // ready for this slot's next launch
                    }
                    __syncwarp();
                    if (k1_hint()) {
                        wait_k1();
                        merge_pieces(u, own, m, l, o);
                    } else {  // K1 still runs: publish the own piece too and merge in drain()
                        publish();
                        if (lane == 0) plist[npark] = u | (int)0x80000000;
                        ++npark;
                        if (npark == NPARK) drain();
                    }
                } else if (designated) {
                    publish();
                    if (lane == 0)
                        asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(unit_count + u) : "memory");
                } else {
                    // one acq_rel arrival by lane 0: release covers the whole warp's stores
                    // (ordered before it by the warp barrier), acquire makes the other pieces'
                    // stores visible to the merging warp (read from L2 with ld.cg)
                    publish();
                    int old = 0;
                    if (lane == 0)
                        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                                     : "=r"(old) : "l"(unit_count + u) : "memory");
                    old = __shfl_sync(0xffffffffu, old, 0);
                    if (old == nseg - 1) {
                        if (lane == 0) unit_count[u] = 0;  // ready for this slot's next launch
                        if (k1_hint()) {
                            wait_k1();
                            merge_pieces(u, own, m, l, o);
                        } else {
                            if (lane == 0) plist[npark] = u | (int)0x80000000;
                            ++npark;
                            if (npark == NPARK) drain();
                        }
                    }
                }
            }
            __syncwarp();
        }
    }
    if (npark > 0) drain();
    K2_TRACE(gw, 6);
    // the launch's last warp resets this layer slot's completion hints
    __syncwarp();
    if (lane == 0) {
        const uint32_t done = atomicAdd(P.k2_done + ls, 1u);
        if (done == (uint32_t)P.nwarps - 1) {
            P.k1_done[ls] = 0;
            P.k2_done[ls] = 0;
        }
    }
    K2_TRACE(gw, 3);
}

template <int D, int G, int kWarps, int kStages>
cudaError_t launch_t(const CUtensorMap *tmk, const CUtensorMap *tmv, const SuffixArgs &a, cudaStream_t s) {
    using S = Shape<D, G, kWarps, kStages>;
    const int smem = S::SMEM;
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
    return cudaLaunchKernelEx(&cfg, kern, *tmk, *tmv, a);
}

}  // namespace

cudaError_t launch_suffix_decode(const CUtensorMap *tmap_k, const CUtensorMap *tmap_v, const PlanDev &p,
                                 const PoolGeom &g, int layer, const void *q, float *out, float *lse,
                                 float scale, cudaStream_t s) {
    SuffixArgs a;
    a.p = p;
    a.layer_blk = (int64_t)layer * g.cap;
    a.q = static_cast<const uint16_t *>(q);
    a.out = out;
    a.lse = lse;
    a.hkv = g.hkv;
    a.hq = g.hq;
    a.qscale = scale * kLog2e;
    a.layer = layer;
    const int G = g.hq / g.hkv;
#define HALO_K2_CASE(DD, GG)                                                                       \
    if (g.d == DD && G == GG)                                                                      \
        return p.k2_warps == kK2WarpsNarrow ? launch_t<DD, GG, kK2WarpsNarrow, kK2StagesNarrow>(tmap_k, tmap_v, a, s) \
                                            : launch_t<DD, GG, kK2WarpsWide, kK2StagesWide>(tmap_k, tmap_v, a, s);
    HALO_K2_CASE(128, 1) HALO_K2_CASE(128, 2) HALO_K2_CASE(128, 4) HALO_K2_CASE(128, 8)
    HALO_K2_CASE(64, 1) HALO_K2_CASE(64, 2) HALO_K2_CASE(64, 4) HALO_K2_CASE(64, 8)
#undef HALO_K2_CASE
    return cudaErrorInvalidValue;
}

}  // namespace halo

// ---------------------------------------------------------------------------------------
// K3 standalone: the LSE merge for plans with no K2 blocks at all (prefill plans whose causal
// parts all ran in K1: every output row is a merge of its K1 partials).  Inside K2 such units
// are latency chains (a warp merges its ~74 units one after another); here one warp merges one
// (request, q-head) row with all its slots' loads in flight together, grid-stride over the rows
// -> HBM-bound.  Same arithmetic as K2's finalize with an empty suffix state (online over the
// slots in ascending order; the first slot sets the reference).
namespace halo {
namespace {

template <int D>
__global__ void __launch_bounds__(256) merge_only_kernel(const PlanDev p, int32_t hq, float *out, float *lse,
                                                           int32_t layer) {
    // K1 (the previous grid) wrote the partials: wait for it before reading them, and let the
    // next layer's K1 start its prologue (it waits for this grid before writing partials)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (blockIdx.x == 0 && threadIdx.x == 0) p.k1_done[layer & 3] = 0;  // K1 is complete: reset the hint
    constexpr int C4 = D / 4;  // float4 chunks per row
    const int lane = threadIdx.x & 31;
    const int64_t rows = (int64_t)p.nreq * hq, slot_stride = rows;
    for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
         row += (int64_t)gridDim.x * (blockDim.x >> 5)) {
        const int nslots = p.req_nslots[row / hq];
        float M = -INFINITY, L = 0.f;
        float4 acc[(C4 + 31) / 32];
#pragma unroll
        for (int k = 0; k < (C4 + 31) / 32; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        // up to kPre slots' loads issued together (one round trip), folded in slot order
        constexpr int kPre = 4, KC = (C4 + 31) / 32;
        float xs[kPre];
        float4 vs[kPre][KC];
#pragma unroll
        for (int sl = 0; sl < kPre; ++sl)
            if (sl < nslots) {
                const int64_t r = sl * slot_stride + row;
                xs[sl] = __ldcg(p.part_lse + r);
#pragma unroll
                for (int k = 0; k < KC; ++k)
                    if (k * 32 + lane < C4) vs[sl][k] = __ldcg(reinterpret_cast<const float4 *>(p.part_o + r * D) + k * 32 + lane);
            }
        for (int sl = 0; sl < nslots; ++sl) {
            const int64_t r = sl * slot_stride + row;
            float x;
            float4 v[KC];
            if (sl < kPre) {
#pragma unroll
                for (int i = 0; i < kPre; ++i)
                    if (i == sl) {
                        x = xs[i];
#pragma unroll
                        for (int k = 0; k < KC; ++k) v[k] = vs[i][k];
                    }
            } else {
                x = __ldcg(p.part_lse + r);
#pragma unroll
                for (int k = 0; k < KC; ++k)
                    if (k * 32 + lane < C4) v[k] = __ldcg(reinterpret_cast<const float4 *>(p.part_o + r * D) + k * 32 + lane);
            }
            x *= kLog2e;
            const float mn = fmaxf(M, x);
            const float al = ptx::ex2(M - mn), w = ptx::ex2(x - mn);
            L = L * al + w;
            M = mn;
#pragma unroll
            for (int k = 0; k < (C4 + 31) / 32; ++k) {
                acc[k].x = fmaf(w, v[k].x, acc[k].x * al);
                acc[k].y = fmaf(w, v[k].y, acc[k].y * al);
                acc[k].z = fmaf(w, v[k].z, acc[k].z * al);
                acc[k].w = fmaf(w, v[k].w, acc[k].w * al);
            }
        }
        const float inv = 1.f / L;
#pragma unroll
        for (int k = 0; k < (C4 + 31) / 32; ++k)
            if (k * 32 + lane < C4)
                reinterpret_cast<float4 *>(out + row * D)[k * 32 + lane] =
                    make_float4(acc[k].x * inv, acc[k].y * inv, acc[k].z * inv, acc[k].w * inv);
        if (lse != nullptr && lane == 0) lse[row] = (M + __log2f(L)) * kLn2;
    }
}

}  // namespace

cudaError_t launch_merge_only(const PlanDev &p, const PoolGeom &g, int layer, float *out, float *lse, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms * 16);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (g.d == 128) return cudaLaunchKernelEx(&cfg, merge_only_kernel<128>, p, g.hq, out, lse, (int32_t)layer);
    if (g.d == 64) return cudaLaunchKernelEx(&cfg, merge_only_kernel<64>, p, g.hq, out, lse, (int32_t)layer);
    return cudaErrorInvalidValue;
}

}  // namespace halo
