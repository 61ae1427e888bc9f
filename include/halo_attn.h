/*
 * halo_attn.h -- C ABI of the B200-native shared-prefix decode-attention library.
 *
 * The hot path behind Halo's KV-cache sharing (arXiv 2509.02121):
 *   - a shared prefix cache: a prefix's K/V is computed once and reused by every later
 *     query with that prefix (§3.3 "Prefix caching");
 *   - the consolidated query-plan DAG makes batched requests share prompt prefixes
 *     (PAPER.md:54 §1, :273 §3.1), which induces a TREE of shared KV segments;
 *   - decode reuses cached key/value tensors and is memory-bound (§2.1,
 *     :341 §3.3), with the decode batch grown to the memory limit (:341);
 *   - KV tensors are the standardised state exchanged at operator boundaries
 *     ("On-the-fly context exchange"); the exchange layout below is
 *     [layer][token][kv_head][head_dim] bf16;
 *   - cache snapshots migrate among GPUs via NVLink under scheduler control
 *     (PAPER.md:337 §3.3, :673 §4.5);
 *   - every optimisation is semantics-preserving: the shared-prefix result equals naive
 *     unshared attention (§2.2 "Exact answers").
 *
 * Only plain C types cross this boundary.  Every `stream` argument is a cudaStream_t
 * passed as void* (NULL = legacy default stream).  Unless stated otherwise, data
 * pointers are DEVICE pointers of the pool's device; entries marked "host or device"
 * accept either (host memory is staged by the library; pinned memory is fastest).
 *
 * Errors: every call returns a halo_status.  Host-side validation finishes before any
 * device work is enqueued; on a non-OK status the library state is unchanged (no partial
 * registration, no leaked blocks).  Asynchronous device faults surface as HALO_ECUDA at
 * the next call that synchronises.  No C++ exception crosses the ABI.  The text of the
 * last error on the calling thread is returned by halo_last_error().
 *
 * Threading: a pool (and its plans) is externally synchronised -- one host thread at a
 * time.  All device work is stream-ordered on the caller's stream.  Blocks given back
 * (request close, truncate, prefix release, MOVE, offload) return to the free list once the
 * work enqueued so far on every stream that used the pool (the 16 most recent; an older one is
 * synchronised before it is forgotten) has passed.
 *
 * Plans: a plan records block ids.  Any call that gives blocks back (the list above) makes
 * every plan built before it stale: halo_decode_run then returns HALO_EBUSY; re-plan
 * (halo_decode_plan with the plan as *inout).  A fetch does not (no plan can contain an
 * offloaded node).
 *
 * Ids: node and request ids are int64, unique and never reused within a pool.
 */
#ifndef HALO_ATTN_H
#define HALO_ATTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HALO_ABI_VERSION 1
#define HALO_BLOCK_TOKENS 16

typedef int32_t halo_status;
enum {
    HALO_OK = 0,
    HALO_EINVAL = 1,        /* bad argument (shape, id kind, null pointer, ...)        */
    HALO_ENOMEM = 2,        /* pool out of blocks, or a device/host allocation failed   */
    HALO_ENOENT = 3,        /* unknown node / request id                                */
    HALO_EBUSY = 4,         /* node still referenced by children or requests            */
    HALO_ECUDA = 5,         /* a CUDA runtime/driver call failed                        */
    HALO_ENCCL = 6,         /* an NCCL call failed, or no communicator                  */
    HALO_EUNSUPPORTED = 7   /* valid but not supported (e.g. compute on a host-only pool) */
};

typedef struct halo_pool_s *halo_pool;
typedef struct halo_plan_s *halo_plan;

/* Text of the last non-OK status raised on this thread ("" if none).  Owned by the
 * library; valid until the next call on this thread. */
const char *halo_last_error(void);
int32_t halo_abi_version(void);

/* ------------------------------------------------------------------ paged KV pool */
/* A pool holds K and V for `num_layers` layers in fixed blocks of 16 tokens.  Device
 * layout of each of K and V (bf16):
 *     [layer][block][kv_head][16][head_dim]
 * so one (block, kv_head) slab is 16*head_dim*2 bytes contiguous (4 KiB at d=128).
 * (Block-level KV management as in vLLM, §4.1 Baselines.)
 * Value domain: any finite bf16 K and V.  (The prefix kernel multiplies V by an exact power
 * of two per tile before its fp16 P.V MMA so that V beyond fp16's range neither overflows nor
 * loses precision; inf / nan inputs propagate.)  The library zero-fills the pool at creation
 * (caller storage included), so never-written slots hold finite values. */
typedef struct {
    int32_t device;          /* CUDA ordinal.  -1 = host-only bookkeeping: no device
                                memory, no launches (used to test allocator/tree/plan on
                                machines without a GPU; compute calls return
                                HALO_EUNSUPPORTED). */
    int32_t num_layers;      /* >= 1 */
    int32_t num_kv_heads;    /* kv heads held by THIS pool (a shard when heads are split) */
    int32_t num_q_heads;     /* q heads served; a multiple g of num_kv_heads; q-head h
                                reads kv head floor(h/g) (reading R3)          */
    int32_t head_dim;        /* 64 or 128 */
    int32_t block_tokens;    /* must be HALO_BLOCK_TOKENS (16) */
    int64_t capacity_blocks; /* blocks per layer; capacity_blocks * num_kv_heads <= 2^27
                                and num_layers * capacity_blocks < 2^31 (EINVAL)      */
    void *k_storage;         /* optional caller-owned device memory for K (and V), each of
                                >= halo_pool_storage_bytes(cfg) bytes, 256-B aligned;
                                NULL => the library allocates (and frees) it.           */
    void *v_storage;
} halo_pool_config;

/* Bytes of ONE of the K or V arrays for this config. */
size_t halo_pool_storage_bytes(const halo_pool_config *cfg);
halo_status halo_pool_create(const halo_pool_config *cfg, halo_pool *out);
/* Frees every node, request and plan resource of the pool.  Plans created on it must be
 * destroyed first (EBUSY otherwise). */
halo_status halo_pool_destroy(halo_pool pool);
halo_status halo_pool_stats(halo_pool pool, int64_t *free_blocks, int64_t *used_blocks);
/* Device base pointers of the K and V arrays (layout above).  For tests and tools. */
halo_status halo_pool_storage(halo_pool pool, void **k, void **v);

/* ------------------------------------------------------------------ prefix nodes */
/* Register an immutable shared prefix segment of `ntok` tokens under `parent` (-1 = a
 * root): the "shared prefix cache" entry of PAPER.md:343.  k, v (host or device):
 * bf16 [num_layers][ntok][num_kv_heads][head_dim] (the exchange layout).  Copies the
 * tokens into freshly allocated blocks on `stream` (tail of the last block zero-filled);
 * the caller may reuse k/v once `stream` has passed this point.  ntok >= 1. */
halo_status halo_prefix_register(halo_pool pool, int64_t parent, int32_t ntok,
                                 const void *k, const void *v, void *stream,
                                 int64_t *node_out);
/* Release a node: EBUSY while it has children or open requests.  Its blocks return to
 * the pool once work already enqueued on the pool's streams has passed. */
halo_status halo_prefix_release(halo_pool pool, int64_t node);
/* Gather a node's tokens out of the pool into k_out, v_out (device): bf16
 * [num_layers][ntok][num_kv_heads][head_dim].  This is the K4 pack kernel. */
halo_status halo_prefix_read(halo_pool pool, int64_t node, void *k_out, void *v_out,
                             void *stream);
/* Introspection: parent, token count, block count, and (if blocks_out != NULL, with room
 * for *nblocks entries) the block ids in token order. */
halo_status halo_node_info(halo_pool pool, int64_t node, int64_t *parent, int32_t *ntok,
                           int32_t *nblocks, int32_t *blocks_out);

/* ------------------------------------------------------------------ requests */
/* Open a decode request under prefix node `leaf` (-1 = no shared prefix).  Its private
 * suffix starts empty and always starts in a fresh block (reading R11). */
halo_status halo_request_open(halo_pool pool, int64_t leaf, int64_t *req_out);
halo_status halo_request_close(halo_pool pool, int64_t req);
halo_status halo_request_info(halo_pool pool, int64_t req, int64_t *leaf, int32_t *suffix_len,
                              int32_t *nblocks);
/* Append ntok[i] >= 0 tokens to the suffix of reqs[i] (reqs and ntok are HOST arrays).
 * k, v (host or device): bf16 [num_layers][sum(ntok)][num_kv_heads][head_dim], requests
 * in the order given.  All-or-nothing: ENOMEM leaves every suffix unchanged.  K5. */
halo_status halo_suffix_append(halo_pool pool, int32_t nreq, const int64_t *reqs,
                               const int32_t *ntok, const void *k, const void *v,
                               void *stream);
/* Drop the last ntok[i] tokens of each suffix (host-only bookkeeping; freed blocks return
 * to the pool after enqueued work passes).  Used to roll back tokens. */
halo_status halo_suffix_truncate(halo_pool pool, int32_t nreq, const int64_t *reqs,
                                 const int32_t *ntok);

/* ------------------------------------------------------------------ decode step */
/* A zero-initialised struct (or NULL) selects every default. */
typedef struct {
    int32_t min_tensor_rows; /* a prefix node runs on the tcgen05 prefix kernel (K1) iff
                                (#requests under it) * g >= this; others are folded into
                                the suffix kernel as ordinary blocks.  <= 0: default 64. */
    int32_t force_splits;    /* > 0: split every K1 node's tokens into this many ranges
                                (tests); 0: the plan chooses (fills the 148 SMs).      */
    int32_t max_splits;      /* cap on splits per node; <= 0: default 16                */
    int32_t k2_chunk_blocks; /* K2 work-queue chunk in 16-token blocks; <= 0: plan chooses */
    int32_t k2_shape;        /* K2 launch shape: 0 = plan chooses, 1 = wide (12 warps x 2
                                ring stages per SM), 2 = narrow (7 warps x 4 stages)    */
    int32_t k2_sms;          /* > 0: K2's schedule and grid use this many SMs; 0 = all    */
    float k1_sm_frac;        /* single-wave K1 beside a dominant K2 may take this fraction
                                of the SMs (K2); 0 = default 0.65, < 0 = off   */
    float k2_early_weight;   /* work weight of K2 warps that start beside K1 (on SMs K1
                                leaves idle); 0 = default (1.2 when the K1 rule applies) */
    int32_t k2_tail_pct;     /* > 0: K2's last k2_tail_pct % of blocks are cut into small
                                pieces that warps claim dynamically once their static share
                                is done; <= 0: off (default: measured slower at C1)        */
    int32_t k2_whole_units;  /* >= 0 (default): with few units per warp and no K1 beside
                                it, K2 runs whole units over the narrow shape (no stream-K
                                pieces; C1 K2 alone 0.83 of HBM); < 0: the wide shape with
                                pieces (0.78-0.80)                                          */
} halo_plan_options;

/* Build (or rebuild in place, when *inout != NULL) the plan of one decode step for the
 * batch reqs[0..nreq) (HOST array, any order).  The plan records the prefix tree of the
 * batch in DFS order (so each node covers a contiguous request range), the K1 tile list,
 * the K2 work list and the partial-slot map, and uploads them on `stream`.  Reuse a plan
 * only on the stream its runs were enqueued on.  Requests with an empty context
 * (no prefix and no suffix token) are EINVAL. */
halo_status halo_decode_plan(halo_pool pool, int32_t nreq, const int64_t *reqs,
                             const halo_plan_options *opt, void *stream, halo_plan *inout);
/* Prefill against cached prefixes (PAPER.md:121 §2.1 prefill; :321 KV-cache reuse discount
 * gamma; :343 shared prefix cache): request reqs[i] has just appended ntok[i] >= 1 prompt
 * tokens (the last ntok[i] tokens of its suffix, K/V already in the pool via
 * halo_suffix_append).  The plan's rows are those tokens, request by request in the given
 * order, tokens in order (sum ntok rows); row t of request i attends to the request's prefix
 * path and to its suffix up to and including that token (causal within the prompt).  Run it
 * with halo_decode_run / halo_decode_layers with q / out / lse rows = the new tokens
 * ([sum ntok][Hq][d]).  The shared-prefix part is K1 on tensor cores over all the tokens of
 * all the requests under a node; the causal suffix part runs in K2 (each token streams the
 * suffix blocks it sees).  EINVAL if ntok[i] is out of [1, suffix length]. */
halo_status halo_prefill_plan(halo_pool pool, int32_t nreq, const int64_t *reqs, const int32_t *ntok,
                              const halo_plan_options *opt, void *stream, halo_plan *inout);
/* Attention of layer `layer` for the planned batch:
 *   q   : bf16 [nreq][num_q_heads][head_dim], rows in the order given to the plan
 *   out : fp32 [nreq][num_q_heads][head_dim]   normalised attention output
 *   lse : fp32 [nreq][num_q_heads] natural-log log-sum-exp of the scaled scores (nullable)
 *   scale <= 0 selects 1/sqrt(head_dim).
 * Enqueues K1 (shared prefixes, tcgen05) then K2 (private suffixes + fused LSE merge, K3).
 * Graph-capturable. */
halo_status halo_decode_run(halo_plan plan, int32_t layer, const void *q, float *out,
                            float *lse, float scale, void *stream);
/* One decode step of the batch, the call a serving loop makes (PAPER.md:341 decode batch;
 * append-then-attend, R4): append ONE token per request (k_new, v_new: bf16
 * [num_layers][nreq][num_kv_heads][head_dim]), (re)plan into *inout (NULL: a new plan, as
 * halo_decode_plan), then attention of every layer (q: bf16 [num_layers][nreq][Hq][d];
 * out: fp32 [num_layers][nreq][Hq][d]; lse nullable fp32 [num_layers][nreq][Hq]).
 * Every buffer may be host (pinned for overlap) or device.  Pipelined per layer: the
 * host->device copies of layer l+1 and the device->host copy of layer l-1 overlap the
 * append + K1 + K2/K3 kernels of layer l (two library-owned copy streams, events).  All
 * work is complete in `stream` order when the call's work on `stream` is.  Errors before
 * any launch (ENOENT, ENOMEM, EINVAL) leave the pool unchanged. */
halo_status halo_decode_step(halo_pool pool, int32_t nreq, const int64_t *reqs, const void *k_new,
                             const void *v_new, const void *q, float *out, float *lse, float scale,
                             const halo_plan_options *opt, void *stream, halo_plan *inout);
/* Run only some stages of halo_decode_run (for per-kernel timing): stage_mask bit 0 = K1
 * (prefix partials), bit 1 = K2+K3 (suffix + merge; reads the partials K1 last wrote for
 * this plan).  halo_decode_run == stage_mask 3. */
halo_status halo_decode_run_stages(halo_plan plan, int32_t layer, int32_t stage_mask,
                                   const void *q, float *out, float *lse, float scale,
                                   void *stream);
/* All layers [0, nlayers) in one call: q (host or device) bf16 [nlayers][nreq][Hq][d],
 * out (host or device) fp32 [nlayers][nreq][Hq][d], lse (nullable, host or device) fp32
 * [nlayers][nreq][Hq].  Host buffers are staged through device scratch on `stream`. */
halo_status halo_decode_layers(halo_plan plan, int32_t nlayers, const void *q, float *out,
                               float *lse, float scale, void *stream);

typedef struct {
    int32_t nreq, num_q_heads, num_kv_heads, head_dim;
    int32_t tensor_nodes;    /* prefix nodes on K1 */
    int32_t folded_nodes;    /* prefix nodes folded into K2 */
    int32_t k1_tiles;        /* K1 CTAs per layer */
    int32_t k2_units;        /* (request, kv head) work units of K2 */
    int32_t max_slots;       /* partial slots per request (max over requests) */
    int32_t k2_warps;        /* K2 launch shape: warps per CTA (12 wide / 7 narrow) */
    int64_t k1_rows;         /* sum over K1 tiles of valid rows x tokens / 128 (bookkeeping) */
    double k1_flops;         /* algorithmic FLOPs per layer: sum_nodes 4*(n_req*g)*L_n*d*Hkv */
    double k1_bytes;         /* algorithmic bytes per layer of K1 (KV once + Q + partials) */
    double k2_bytes;         /* algorithmic bytes per layer of K2+K3 */
    double unshared_bytes;   /* KV bytes per layer an unshared decode would read */
} halo_plan_info;
halo_status halo_plan_get_info(halo_plan plan, halo_plan_info *info);
/* Copy one of the plan's host arrays out (tests): which = 0 request DFS order (int32
 * caller indices), 1 K1 tiles (int32 x 8 each: req_off, nrows, kv_head, tok_begin,
 * tok_end, blk_off, slot, node_index), 2 per-request slot counts (int32), 3 K2 request
 * order (int32), 4 per-request K2 block CSR offsets (int32, nreq+1), 5 K2 block entries
 * (uint32: block | (ntok-1) << 27), and the K2 schedule: 6 unit block offsets (nunits+1),
 * 7/8 first/end unit of each chunk, 9 pieces per unit, 10 chunk block bounds (nchunks+1),
 * all int32.  *n receives the element count; copies at
 * most cap. */
halo_status halo_plan_export(halo_plan plan, int32_t which, void *dst, int64_t cap,
                             int64_t *n);
halo_status halo_plan_destroy(halo_plan plan);

/* ------------------------------------------------------------------ migration */
/* KV-block migration between GPUs: "cache snapshots can be migrated directly among GPUs via
 * NVLink ... under scheduler control" (PAPER.md:337 §3.3; NVLink, :673 §4.5), overlapped
 * with decode attention (PAPER.md:9 abstract, :59 §1).  NCCL point-to-point over
 * NVLink/NVSwitch is used ONLY here.  The 128-B ncclUniqueId is created on one rank
 * (halo_comm_unique_id) and broadcast by the caller (torch.distributed).
 *
 * Wire format (both peers derive it from the node's token count and the pool geometry, which
 * must agree: num_layers, num_kv_heads, head_dim): the node's blocks flattened layer-major
 * into items j = layer * nblk + b (nblk = ceil(ntok/16)); item j is the whole (layer, block)
 * slab of K then of V, [hkv][16][d] bf16 each (partial last block: its zero tail moves too,
 * so every destination slab is bit-identical to its source slab).  A transfer is cut into
 * chunks of chunk_items = max(1, chunk_bytes / item_bytes) items; chunk c of every transfer
 * of one exchange call moves in round c, each round ONE ncclGroupStart/End (so a pair of
 * ranks that send to each other in the same call cannot deadlock), double-buffered: the K4
 * pack of round c+1 and the K4 unpack of round c-1 (on `stream`) overlap the NCCL transfer of
 * round c (on a library side stream). */
typedef struct {
    int32_t max_ctas;     /* NCCL maxCTAs of the communicator (bounds the SMs NCCL takes from
                             decode while a migration runs); <= 0: NCCL's default          */
    int32_t copy_ctas;    /* CTAs of the K4 pack / unpack kernels; <= 0: 8 x SM count       */
    int64_t chunk_bytes;  /* bytes per transfer per round (K+V); <= 0: 32 MiB.  MUST be equal
                             on every rank (it fixes the wire chunking).                    */
} halo_comm_config;

halo_status halo_comm_unique_id(void *id_out /* 128 bytes */);
/* Create the pool's communicator (collective over the nranks ranks: every rank calls it with
 * the same id).  nranks == 1 is a valid self-loop communicator (loopback migration on one
 * GPU: the exact pack -> NCCL -> unpack -> register pipeline).  cfg nullable (defaults).
 * EBUSY if the pool already has one; ENCCL if libnccl.so.2 is unavailable or NCCL fails. */
halo_status halo_comm_init(halo_pool pool, const void *id /* 128 bytes */, int32_t nranks,
                           int32_t rank);
halo_status halo_comm_init_config(halo_pool pool, const void *id /* 128 bytes */, int32_t nranks,
                                  int32_t rank, const halo_comm_config *cfg);

typedef struct {
    int64_t node;     /* node to send (device-resident)                                       */
    int32_t peer;     /* destination rank; may be this rank (self loop, matched by a recv of
                         the same call)                                                       */
    int32_t mode;     /* 0 = MOVE (node released once the transfer has passed; EBUSY if it has
                         children or open requests), 1 = COPY                                  */
} halo_migrate_send_op;

typedef struct {
    int64_t parent;   /* register the received node under this node (-1 = a root)           */
    int32_t peer;     /* source rank; may be this rank                                         */
    int32_t ntok;     /* tokens of the node being received (>= 1; the sender's ntok)           */
} halo_migrate_recv_op;

/* One batch of migrations on this rank: send sends[0..nsend) and receive recvs[0..nrecv)
 * (HOST arrays; either count may be 0).  Every rank taking part calls it at the same point of
 * its NCCL program.  Pairing: the k-th send of rank a to peer b matches the k-th recv of rank
 * b from peer a (NCCL point-to-point order), with equal token counts -- the caller's
 * scheduler guarantees this (relocation.rank_actions); for self-loop ops the library checks
 * it (EINVAL).  Received nodes are registered in recv order; their ids go to nodes_out[nrecv]
 * (HOST).  Validation (ids, peers, modes, MOVE of a referenced or twice-listed node, parents,
 * and the allocation of every destination block: ENOMEM) completes before any device work;
 * on error nothing changes.  Stream-ordered: pack and unpack kernels run on `stream` (pass a
 * side stream to overlap decode on another one), NCCL on a library stream; on return `stream`
 * is ordered after every send and receive of the call.  The received nodes may be used (plans,
 * requests) immediately in `stream` order.  Sources of MOVEs are released (their blocks return
 * to the pool once `stream` has passed this call). */
halo_status halo_migrate_exchange(halo_pool pool, int32_t nsend, const halo_migrate_send_op *sends,
                                  int32_t nrecv, const halo_migrate_recv_op *recvs, void *stream,
                                  int64_t *nodes_out);
/* One send (== halo_migrate_exchange with one send op).  dst_rank != this rank. */
halo_status halo_migrate_send(halo_pool pool, int64_t node, int32_t dst_rank, int32_t mode,
                              void *stream);
/* One receive (== halo_migrate_exchange with one recv op).  src_rank != this rank. */
halo_status halo_migrate_recv(halo_pool pool, int32_t src_rank, int64_t parent, int32_t ntok,
                              void *stream, int64_t *node_out);
/* Same-device relocation ("cache snapshots ... migrated"): copy `node` of
 * `src` into fresh blocks of `dst` (which may be the same pool; same device and KV
 * geometry, EINVAL otherwise) under `parent_dst`.  One whole-block pool-to-pool copy
 * kernel: a (layer, block) of all heads is contiguous on both sides.  Stream-ordered on
 * `stream`; ENOMEM leaves dst unchanged. */
halo_status halo_prefix_clone(halo_pool src, int64_t node, halo_pool dst, int64_t parent_dst,
                              void *stream, int64_t *node_out);

/* ------------------------------------------------------------------ host paging
 * The executor's I/O subsystem "asynchronously pages activation caches between GPU and host
 * memory ... prefetch upcoming caches and evict stale ones under the scheduler's control"
 * (PAPER.md:350 §3.3; snapshots "offloaded to host memory under scheduler control", :337).
 * A prefix node is either device-resident (its blocks in the pool) or offloaded (its KV in
 * blocks of a pinned host arena, same [layer][block][head][16][d] layout).  Offload / fetch
 * are stream-ordered copies on the copy engines (one cudaMemcpyAsync per run of consecutive
 * blocks per layer); the blocks they give up return to their free lists once the enqueued
 * copy has passed.  Plans that read an offloaded node fail with HALO_EBUSY; a plan built
 * before an offload is stale and halo_decode_run returns HALO_EBUSY (re-plan). */

/* (Re)allocate the pinned host arena: host_blocks blocks x all layers x K and V.  EBUSY while
 * nodes are offloaded; ENOMEM (arena cleared) if the pinned allocation fails.  On a host-only
 * pool (device -1) this is bookkeeping only (tests). */
halo_status halo_pool_host_reserve(halo_pool pool, int64_t host_blocks);
/* Evict: copy the node's blocks to fresh host-arena blocks on `stream`, then release its
 * device blocks.  ENOENT unknown node; EINVAL already offloaded; EUNSUPPORTED no arena;
 * ENOMEM arena full (nothing changes). */
halo_status halo_prefix_offload(halo_pool pool, int64_t node, void *stream);
/* Prefetch: copy an offloaded node back into fresh device blocks on `stream` (same node id,
 * tree position and requests).  EINVAL if not offloaded; ENOMEM pool full (nothing
 * changes). */
halo_status halo_prefix_fetch(halo_pool pool, int64_t node, void *stream);
/* Background prefetch ("prefetch upcoming caches ... just in time"): fetch, on
 * `stream` (typically a copy stream beside the decode stream), every offloaded node on the
 * prefix paths of reqs[0..nreq) (HOST array), parents first.  Each fetch records an event;
 * plans built afterwards on any stream (and halo_prefix_read / clone / migrate of the node) wait
 * for it, so the next step's plan can be built right away while the copies overlap the current
 * step.  *n_fetched (nullable) = nodes fetched.  ENOMEM: the fetches made so far stay (evict
 * with halo_pool_evict_lru first). */
halo_status halo_pool_prefetch(halo_pool pool, int32_t nreq, const int64_t *reqs, void *stream,
                               int32_t *n_fetched);
/* on_device: 1 resident, 0 offloaded; last_use: LRU clock of the last plan that read it. */
halo_status halo_node_residency(halo_pool pool, int64_t node, int32_t *on_device, uint64_t *last_use);
/* LRU eviction policy: offload device-resident nodes in increasing last_use (ties: lower id),
 * never one read by the most recent plan, until free + pending-free device blocks >=
 * want_free.  *n_evicted = nodes offloaded.  ENOMEM if the target cannot be reached (the
 * evictions made so far stay). */
halo_status halo_pool_evict_lru(halo_pool pool, int64_t want_free, void *stream, int32_t *n_evicted);

/* ------------------------------------------------------------------ relocation planner
 * Cost-model placement of prefix groups on workers (GPUs): PAPER.md Alg. 1 (§3.2, "Beam
 * Search with Incremental Cost") with the cost functions of §3.2 "Cost Functions"
 * (PAPER.md:315-332).  An item is one prefix group: a prefix tree (its nodes' KV) with the
 * decode requests under it -- the operator whose placement decides where its KV lives.
 * Host-only (no device work); the caller executes the returned moves with
 * halo_migrate_send/recv (another GPU), halo_prefix_clone (same GPU) or halo_prefix_fetch
 * (host arena).  Readings (DESIGN.md §5 "Relocation planner"):
 *   - e_v = exec_s, the item's decode-attention time on one worker;
 *   - p_v = context preparation on worker d: 0 if d == home, kv_bytes / link_bytes_per_s if
 *     another worker holds the KV (relocation over NVLink), prep_s if none does (host
 *     fetch or prefill);  gamma_v = sigma_v = lambda_v = 1 (e_v already counts prefix
 *     sharing; no model weights or retrieval state move on this path);
 *   - C_a^d = sum_{v on d} e_v / k_v^beta + p_v(d);  C_a = max_d C_a^d;
 *     C_r = (sum of e_v over unassigned items) / m^beta;  Cost = C_a + C_r;
 *   - V_r = the ops_per_iter unassigned items of largest e_v (ties: lower index) -- the
 *     paper's "top-|D| ready operators"; items are independent (no DAG edges between
 *     prefix groups), so every unassigned item is ready;
 *   - replication over k > 1 workers (queries partitioned over replicas) is offered only
 *     when fewer items remain unassigned than there are workers and e_v >= (sum of all
 *     e_v) / workers (the paper's conditions (i), (ii)); the replica set is the home worker
 *     (if any) plus the least-loaded other workers of the partial assignment;
 *   - ties between equal-cost candidates: the lexicographically smaller assignment. */
typedef struct {
    double exec_s;         /* e_v >= 0: decode-attention seconds on one worker          */
    double kv_bytes;       /* bytes one relocation of the item's KV moves (>= 0)        */
    double prep_s;         /* p_v when no worker holds the KV (home == -1), >= 0        */
    int32_t home;          /* worker holding the KV now, or -1                          */
    int32_t max_replicas;  /* >= 1; 1 = single-assigned                                 */
} halo_place_item;

typedef struct {
    int32_t workers;          /* m = |D|, 1..64                                          */
    int32_t beam_width;       /* w >= 1                                                  */
    int32_t ops_per_iter;     /* |V_r| cap per iteration, 1..workers                     */
    int32_t reserved;
    double beta;              /* parallelism decay, >= 0                                 */
    double link_bytes_per_s;  /* measured relocation rate, > 0                           */
} halo_place_config;

typedef struct {
    int32_t item;             /* index into items                                        */
    int32_t src;              /* worker sending the KV; -1 = prepare from host / prefill */
    int32_t dst;              /* worker receiving it                                     */
    int32_t mode;             /* 0 = MOVE (src releases after), 1 = COPY                 */
    double seconds;           /* the p_v this move was costed at                         */
} halo_place_move;

/* Run the beam search.  items: HOST array of n >= 1.  Outputs (HOST):
 *   worker_mask[n]  bit d set <=> item placed on worker d (popcount = its replicas);
 *   load[workers]   (nullable) final C_a^d;   *cost: final Cost (= C_a, nothing unassigned);
 *   moves (nullable, room for move_cap) and *n_moves: the relocations that realise the
 *   placement -- for an item with home h >= 0, one transfer h -> d per placed worker d != h,
 *   COPY except the last when h is not in the placement (MOVE); for home -1, one prepare
 *   (src -1, COPY) per placed worker.  Moves are ordered by item, then worker.
 * EINVAL on a bad argument or when one iteration would enumerate more than 2^20
 * candidates; ENOMEM if move_cap is too small (*n_moves still receives the count). */
halo_status halo_place_groups(const halo_place_config *cfg, int32_t n, const halo_place_item *items,
                              uint64_t *worker_mask, double *load, double *cost,
                              halo_place_move *moves, int32_t move_cap, int32_t *n_moves);

#ifdef __cplusplus
}
#endif
#endif /* HALO_ATTN_H */
