// Host runtime state of libhalo_attn (pool, prefix tree, requests, plans).  Private.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/halo_attn.h"
#include "halo_internal.h"

typedef struct ncclComm *ncclComm_t;

namespace halo {

struct Node {
    int64_t parent = -1;
    int32_t ntok = 0;
    std::vector<int32_t> blocks;       // device blocks (empty while offloaded)
    int32_t children = 0;
    int32_t requests = 0;
    bool on_host = false;              // offloaded: KV lives in host_blocks of the host arena
    std::vector<int32_t> host_blocks;
    uint64_t last_use = 0;             // plan tick of the last plan that read the node (LRU)
    cudaEvent_t ready = nullptr;       // recorded after a fetch's device writes (background
                                       // prefetch): plans / reads of the node wait on it
};

struct Request {
    int64_t leaf = -1;
    int32_t len = 0;  // suffix tokens
    std::vector<int32_t> blocks;
};

struct PendingFree {
    std::vector<cudaEvent_t> events;
    std::vector<int32_t> blocks;
};

struct StreamFence {
    cudaStream_t stream;
    uint64_t last_use;
};

// Ring of pinned host staging buffers for small per-step uploads (plan arrays, slot lists):
// an H2D copy from pinned memory is truly asynchronous (a pageable one makes the host wait for
// the DMA, e.g. behind a large fetch on a copy stream), so the host can build the next step's
// plan while the GPU still runs this one.  acquire() waits for the copy that last used the
// buffer (kPinBufs uploads ago), commit() enqueues the copy and records the buffer's event.
constexpr int kPinBufs = 4;
struct PinRing {
    void *buf[kPinBufs] = {};
    size_t cap[kPinBufs] = {};
    cudaEvent_t ev[kPinBufs] = {};
    bool used[kPinBufs] = {};
    int cur = 0;
    void *acquire(size_t bytes);                                   // nullptr on failure
    cudaError_t commit(void *dst, size_t bytes, cudaStream_t s);   // copies buf[cur] -> dst
    void release();
};

inline void *PinRing::acquire(size_t bytes) {
    cur = (cur + 1) % kPinBufs;
    if (used[cur] && ev[cur]) cudaEventSynchronize(ev[cur]);
    if (!ev[cur] && cudaEventCreateWithFlags(&ev[cur], cudaEventDisableTiming) != cudaSuccess) return nullptr;
    if (cap[cur] < bytes) {
        if (buf[cur]) cudaFreeHost(buf[cur]);
        buf[cur] = nullptr;
        cap[cur] = 0;
        const size_t c = (bytes + bytes / 2 + 4096 + 15) / 16 * 16;
        if (cudaHostAlloc(&buf[cur], c, cudaHostAllocMapped) != cudaSuccess) return nullptr;
        cap[cur] = c;
    }
    return buf[cur];
}

inline cudaError_t PinRing::commit(void *dst, size_t bytes, cudaStream_t s) {
    // SM copy from the mapped buffer (unified addressing: the host pointer is valid on the
    // device): never queued behind another stream's copy-engine transfer
    cudaError_t e = bytes ? launch_h2d_small(buf[cur], dst, bytes, s) : cudaSuccess;
    if (e == cudaSuccess) e = cudaEventRecord(ev[cur], s);
    used[cur] = (e == cudaSuccess);
    return e;
}

inline void PinRing::release() {
    for (int i = 0; i < kPinBufs; ++i) {
        if (ev[i]) cudaEventSynchronize(ev[i]);
        if (buf[i]) cudaFreeHost(buf[i]);
        if (ev[i]) cudaEventDestroy(ev[i]);
        buf[i] = nullptr;
        ev[i] = nullptr;
        cap[i] = 0;
        used[i] = false;
    }
}

// Set the calling thread's halo_last_error() text (for ABI entry points outside runtime.cu).
halo_status report_error(halo_status st, const char *msg);

}  // namespace halo

struct halo_pool_s {
    halo_pool_config cfg{};
    halo::PoolGeom geom{};
    bool host_only = false;
    int num_sms = 148;
    void *k = nullptr, *v = nullptr;
    bool own_storage = false;
    std::vector<int32_t> free_list;  // stack: back() is the next block handed out
    std::vector<uint32_t> blk_epoch; // allocation epoch of each block (V-table tag)
    uint32_t epoch = 0;              // incremented per allocation
    std::vector<halo::PendingFree> pending;
    std::vector<cudaEvent_t> event_cache;
    std::vector<halo::StreamFence> streams;  // streams that enqueued work on this pool
    uint64_t use_clock = 0;
    std::unordered_map<int64_t, halo::Node> nodes;
    std::unordered_map<int64_t, halo::Request> requests;
    int64_t next_id = 1;
    int32_t plans_alive = 0;
    // host paging: pinned arena [layer][host block][head][16][d] x K, V
    void *hk = nullptr, *hv = nullptr;
    int64_t host_cap = 0;
    std::vector<int32_t> host_free;
    std::vector<halo::PendingFree> host_pending;
    uint64_t plan_tick = 0;     // incremented per plan build (LRU clock)
    halo::PinRing pin_up;       // pinned staging of the pool's small uploads (slot / block lists)
    uint64_t layout_gen = 0;    // incremented when a node's blocks move (offload / fetch)
    CUtensorMap tmap_k{}, tmap_v{};      // box: one 16-token block x 64 d
    CUtensorMap tmap_k8{}, tmap_v8{};    // box: 8 consecutive blocks (128 tokens) x 64 d
    // migration
    ncclComm_t comm = nullptr;
    int32_t nranks = 0, rank = -1;
    cudaStream_t side = nullptr;
    void *mig_buf = nullptr;
    size_t mig_cap = 0;
    cudaEvent_t mig_ev[4] = {nullptr, nullptr, nullptr, nullptr};  // packed[2], transferred[2]
    cudaEvent_t mig_done = nullptr;  // last use of mig_buf (end of the last exchange)
    halo_comm_config mig_cfg{};
};

struct halo_plan_s {
    halo_pool pool = nullptr;
    int32_t nreq = 0;
    halo_plan_options opt{};
    std::vector<int32_t> req_order, node_blocks, unit_req, req_blk_off, req_nslots;
    std::vector<int32_t> unit_boff, chunk_lo, chunk_u0, chunk_u1, unit_chunk0, unit_nseg, unit_seg;
    int32_t nseg_total = 0;
    int32_t dyn_first = 0;  // first dynamically claimed K2 chunk (== nchunks: none)
    // equal-share K2 schedule for K2 launched alone (co-schedule weights off)
    std::vector<int32_t> alt_chunk_info, alt_unit_meta;
    std::vector<int32_t> item_unit, item_chunk;  // planner scratch (item -> unit / chunk maps)
    int32_t alt_nchunks = 0, alt_nseg_total = 0;
    int32_t alt_k2_warps = 0;  // launch shape of the K2-alone schedule
    int32_t k2_warps = halo::kK2WarpsWide;
    bool k2_early = false;  // K1 split count lowered so K2's first CTAs stream beside K1
    double k2_early_w = 1.0;  // the co-schedule model's work weight of those CTAs
    std::vector<uint32_t> req_blk;
    std::vector<uint32_t> k2_ent;     // [Btot][2] K2 block descriptors (PlanDev::k2_ent)
    std::vector<int32_t> unit_meta;   // [U][8] K2 unit metadata (PlanDev::unit_meta)
    std::vector<int32_t> chunk_info;  // [NC][4] K2 chunk bounds + unit range (PlanDev::chunk_info)
    std::vector<int32_t> tile_aux;    // [ntiles][4] K1 shortcuts (PlanDev::tile_aux)
    std::vector<halo::PrefixTile> tiles;
    halo_plan_info info{};
    uint64_t layout_gen = 0;    // pool layout generation the plan was built against
    std::vector<uint8_t> host_buf;   // host-only pools
    halo::PinRing pin_plan, pin_slots;
    void *dbuf = nullptr;
    size_t dbuf_cap = 0;
    float *part = nullptr;
    size_t part_cap = 0;
    float *segbuf = nullptr;   // stream-K scratch (seg_o | seg_ml)
    size_t seg_cap = 0;
    int32_t *counters = nullptr;
    size_t counter_cap = 0;
    // K1's TMA map of the q rows (encoded per q buffer; reused while q and nreq are unchanged)
    CUtensorMap tmap_q{};
    const void *tmap_q_ptr = nullptr;
    int32_t tmap_q_nreq = -1;
    bool tmap_q_ok = false;
    halo::PlanDev dev{};
    std::vector<cudaEvent_t> waits;   // fetch events of the plan's nodes (waited at upload)
    // staging for halo_decode_layers with host buffers
    void *q_stage = nullptr;
    size_t q_stage_cap = 0;
    float *o_stage = nullptr;
    size_t o_stage_cap = 0;
    float *l_stage = nullptr;
    size_t l_stage_cap = 0;
    // halo_decode_step: copy streams, per-layer events and the appended token's K/V staging
    cudaStream_t h2d = nullptr, d2h = nullptr;
    std::vector<cudaEvent_t> ev_in, ev_out;
    cudaEvent_t ev_step = nullptr, ev_copied = nullptr;
    // halo_decode_step's input staging is double-buffered (parity e2e_par): ev_used[b] marks
    // the end of the compute that last read buffer b, which the next upload into b waits for
    cudaEvent_t ev_used[2] = {nullptr, nullptr};
    bool ev_used_rec[2] = {false, false};
    int e2e_par = 0;
    void *kv_stage = nullptr;
    size_t kv_stage_cap = 0;
    int32_t *slot_stage = nullptr;
    size_t slot_stage_cap = 0;
};
