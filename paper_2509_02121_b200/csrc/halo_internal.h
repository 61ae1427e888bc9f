// Internal declarations shared by the host runtime and the kernels of libhalo_attn.
// (Product code only; the oracle shares nothing with this file.)
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace halo {

constexpr int kBlockTok = 16;       // tokens per KV block
constexpr int kK1Rows = 256;        // K1 tile rows (two UMMA M=128 sub-tiles)
constexpr int kK1Tok = 128;         // K1 tokens per n-tile (UMMA N of S, K of P.V)
constexpr int kK1MaxTileTok = 4096;  // max token range of one K1 tile (split-N above this; bounded by smem)
// K2 launch shapes (one CTA per SM): "wide" = 12 warps x 2 ring stages (many units per warp:
// best latency hiding), "narrow" = 7 warps x 4 stages (chosen by the planner when units are
// few per warp and whole units divide evenly over 7 warps per SM: no stream-K pieces).
constexpr int kK2WarpsWide = 12, kK2StagesWide = 2;
constexpr int kK2WarpsNarrow = 7, kK2StagesNarrow = 4;
constexpr int kK2HeadPad = 8;       // K2's MMA N dimension: the g q-heads of a unit padded to 8
constexpr int kBlkCountShift = 27;  // K2 block entry: block | (ntok-1) << 27 (| unit start << 31)
constexpr uint32_t kBlkMask = (1u << kBlkCountShift) - 1;

// One K1 work tile: rows [row0, row0+nrows) of node n's (request x q-head-in-group) row
// space for kv head `kv_head`, tokens [tok_begin, tok_end) of the node.
struct PrefixTile {
    int32_t req_off;    // index into req_order of the tile's first request
    int32_t nrows;      // valid rows (<= 128)
    int32_t kv_head;
    int32_t tok_begin;  // multiple of 128
    int32_t tok_end;
    int32_t blk_off;    // index into node_blocks of the node's block 0
    int32_t slot;       // partial slot written by this tile
    int32_t node;       // plan-local node index (diagnostics)
};
static_assert(sizeof(PrefixTile) == 32, "PrefixTile is exported as int32 x 8");

// Device view of a plan (all pointers into one device buffer).
struct PlanDev {
    const PrefixTile *tiles;
    const int4 *tile_aux;        // [ntiles] {caller index of the tile's first request if its
                                 //  requests are consecutive else -1, pool block of its first
                                 //  token if its blocks are consecutive else -1, -, -}
    const int32_t *req_order;    // caller indices, DFS order
    const int32_t *node_blocks;  // block ids of K1 nodes
    const int32_t *unit_req;     // K2 request order (caller indices, LPT)
    const int32_t *req_blk_off;  // [nreq+1] CSR into req_blk, by caller index
    const uint32_t *req_blk;     // block | (ntok-1) << 27
    const int32_t *req_nslots;   // [nreq]
    float *part_o;               // [max_slots][nreq][Hq][D]
    float *part_lse;             // [max_slots][nreq][Hq]
    // K2 schedule: unit u = (request unit_req[u / hkv], kv head u % hkv) covers global block
    // indices [unit_boff[u], unit_boff[u+1]).  The sequence is cut into chunks
    // [chunk_lo[c], chunk_lo[c+1]); warp w processes chunks w, w + nwarps, ... (static);
    // chunk c visits units [chunk_u0[c], chunk_u1[c]).  A unit cut by chunk boundaries
    // writes nseg partial states (slots unit_seg..) merged by the last arriving piece.
    // k2_ent[x] describes global block x: {slab | (ntok-1) << 27 | unit start << 31,
    // q group row | shared << 31}, slab = pool block * hkv + kv head, q group row =
    // request * hkv + head, shared = the block belongs to a folded prefix node (L2 policy).
    // unit_meta[2u], [2u+1] = {boff_begin, boff_end, request, kv head},
    //                         {nslots, nseg, first seg slot, first chunk}.
    const uint2 *k2_ent;         // [nblocks]
    const int4 *chunk_info;      // [nchunks] {chunk_lo[c], chunk_lo[c+1], chunk_u0[c], chunk_u1[c]}
    const int4 *unit_meta;       // [2 * nunits]
    const int32_t *unit_boff;    // [nunits + 1]
    const int32_t *chunk_lo;     // [nchunks + 1]
    const int32_t *unit_chunk0;  // [nunits] first chunk visiting the unit
    const int32_t *chunk_u0;     // [nchunks]
    const int32_t *chunk_u1;     // [nchunks]
    const int32_t *unit_nseg;    // [nunits]
    const int32_t *unit_seg;     // [nunits] first scratch slot (-1 if nseg == 1)
    int32_t *unit_count;         // [nunits] arrival counters (zero between launches)
    float *seg_o;                // [nseg_total][8 heads x D] unnormalised o (base-2 state), K2 fragment layout
    float *seg_ml;               // [nseg_total][8][2]  (m, l) per head
    int32_t ntiles, nreq, nunits, max_slots, nwarps, nchunks, nblocks;
    int32_t k2_warps;            // K2 warps per CTA: kK2WarpsWide or kK2WarpsNarrow
    // static-then-dynamic K2 schedule: warp w streams static chunk w, then claims chunks
    // dyn_first, dyn_first + 1, ... from dyn_counter[layer % 4] (the last claimant resets it);
    // dyn_first == nchunks: static round-robin (warp w takes chunks w, w + nwarps, ...)
    int32_t dyn_first;
    int32_t *dyn_counter;
    // K1 -> K2 completion hint (per layer slot layer % 4): every K1 CTA adds 1 to
    // k1_done[slot] when its partials are written (release); K2 reads it (acquire) to decide
    // whether a finished unit can merge now or is parked until K1 completes; K2's last warp
    // (k2_done) resets both.  Correctness never rests on it (K2 still calls
    // griddepcontrol.wait before any output write).
    uint32_t *k1_done;           // [4]
    uint32_t *k2_done;           // [4]
    // K2 scratch per layer slot (a K2 launch may overlap the previous layer's): stream-K
    // pieces, unit arrival counters and parked unit states are at slot * stride.
    int64_t seg_slot_stride;     // floats between the slots of seg_o (seg_ml likewise, /D*2)
    int32_t count_slot_stride;   // ints between the slots of unit_count
    float *park;                 // [4][nunits][g * (D + 2)]: o (fragment layout), then (m, l) per head
    // equal-share schedule used when K2 is launched without K1 right before it (0: none)
    int32_t alt_nchunks;
    const int4 *alt_chunk_info;
    const int4 *alt_unit_meta;
};

struct PoolGeom {
    int32_t layers, hkv, hq, d;
    int64_t cap;  // blocks per layer
    // V magnitude table [layer][block]: (allocation epoch of the block << 16) | bf16 bits of
    // max |V| over the block's written tokens (all kv heads).  Writers of a block store or
    // atomicMax with the block's epoch, so entries left by a previous owner lose to the
    // current owner's first write.  Read by K1 to pick its per-tile fp16 scale for V.
    uint64_t *vmax;
};
__host__ __device__ inline uint64_t vmax_entry(uint32_t epoch, uint32_t maxbits) {
    return ((uint64_t)epoch << 16) | (maxbits & 0xffffu);
}

// ---- launchers (kernels_*.cu) ----
// K1: tcgen05/TMEM prefix attention -> normalised fp32 partials + lse (natural log).
// tmap_q (nullable): 3-D map {d, q head, request} of q with box {64, g, 128/g}, 128-B
// swizzle -- tiles whose requests are consecutive load their Q rows with it (TMA).
cudaError_t launch_prefix_attn(const CUtensorMap *tmap_k, const CUtensorMap *tmap_v,
                               const CUtensorMap *tmap_k8, const CUtensorMap *tmap_v8,
                               const CUtensorMap *tmap_q, const PlanDev &p, const PoolGeom &g,
                               int layer, const void *q, float scale, cudaStream_t s);
// K2+K3: paged-suffix decode with the fused log-sum-exp merge of the K1 partials.  K/V slabs
// arrive by TMA through the pool's one-block tensor maps (tmap_k / tmap_v, 128-B swizzle).
// K3 alone (plans with no K2 blocks: every row a merge of its K1 partials).
cudaError_t launch_merge_only(const PlanDev &p, const PoolGeom &g, int layer, float *out, float *lse,
                              cudaStream_t s);
cudaError_t launch_suffix_decode(const CUtensorMap *tmap_k, const CUtensorMap *tmap_v, const PlanDev &p,
                                 const PoolGeom &g, int layer, const void *q, float *out, float *lse,
                                 float scale, cudaStream_t s);
// K5 / K4-unpack: rows src[layer][i][head][:] -> pool slot slots[i] (i < n_copy); slots
// [n_copy, n_copy+n_zero) are zero-filled.  src has `src_rows` rows per layer.
// tags[i] (nullable: no V-table update) = allocation epoch of slot i's block.
cudaError_t launch_kv_scatter(const PoolGeom &g, void *pool_k, void *pool_v, const void *src_k,
                              const void *src_v, int64_t src_rows, const int32_t *slots,
                              const uint32_t *tags, int64_t n_copy, int64_t n_zero, int layer_begin,
                              int layer_end, int num_sms, cudaStream_t s);
// K4 pack: pool slot slots[i] -> dst[layer - layer_begin][i][head][:], i < n.
cudaError_t launch_kv_gather(const PoolGeom &g, const void *pool_k, const void *pool_v,
                             void *dst_k, void *dst_v, const int32_t *slots, int64_t n,
                             int layer_begin, int layer_end, int num_sms, cudaStream_t s);

// Same-device relocation: pool block pairs[2i] -> destination block pairs[2i+1], all
// layers in [layer_begin, layer_end), K and V (whole blocks: a partial block's zero tail
// is copied as well).
// dst_tags[i] = allocation epoch of destination block pairs[2i+1] (its V-table entry is the
// source entry's max with this epoch).
cudaError_t launch_kv_copy_blocks(const PoolGeom &sg, const void *src_k, const void *src_v,
                                  const PoolGeom &dg, void *dst_k, void *dst_v,
                                  const int32_t *pairs, const uint32_t *dst_tags, int32_t nblk,
                                  int layer_begin, int layer_end, int num_sms, cudaStream_t s);
// V-table entries of blocks[0..nblk) x layers [0, layers) recomputed from the pool's V (after a
// copy-engine write, e.g. a host-arena fetch); tags[i] = epoch of blocks[i].
cudaError_t launch_kv_vmax(const PoolGeom &g, const void *pool_v, const int32_t *blocks,
                           const uint32_t *tags, int32_t nblk, int num_sms, cudaStream_t s);

// Migration K4 pack (to_pool = false) / unpack (true), block-granular: items
// [item_begin, item_end) of the node's flattened [layer][block] list (layer = j / nblk,
// pool block blocks[j % nblk]); wire layout [item][K|V][hkv][16][d] bf16.  At most max_ctas
// CTAs of 256 threads (bounded so a migration can run beside decode).
// Unpack also writes the V-table entries of the blocks it fills (tags[j % nblk] = epoch).
cudaError_t launch_kv_runs(const PoolGeom &g, void *pool_k, void *pool_v, void *buf,
                           const int32_t *blocks, const uint32_t *tags, int32_t nblk,
                           int64_t item_begin, int64_t item_end, bool to_pool, int max_ctas,
                           cudaStream_t s);

// Host -> device copy of `bytes` by the SMs from MAPPED pinned memory (both 16-B aligned).
cudaError_t launch_h2d_small(const void *mapped_src, void *dst, size_t bytes, cudaStream_t s);

}  // namespace halo
