// Host runtime + C ABI of libhalo_attn: paged KV pool, prefix-node registry, requests,
// the decode-step planner, and NCCL migration.  See include/halo_attn.h for the contract
// and DESIGN.md for the design.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <new>

#include "runtime.h"

using namespace halo;

namespace {

thread_local std::string g_err;

halo_status fail(halo_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

}  // namespace

namespace halo {
halo_status report_error(halo_status st, const char *msg) {
    g_err = msg;
    return st;
}
}  // namespace halo

namespace {

#define HALO_CUDA(expr)                                                                       \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(HALO_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(e_));         \
    } while (0)

#define HALO_NCCL(expr)                                                                       \
    do {                                                                                      \
        if (!nccl().ok) return fail(HALO_ENCCL, "libnccl.so.2 not available");               \
        ncclResult_t r_ = (expr);                                                             \
        if (r_ != ncclSuccess)                                                                \
            return fail(HALO_ENCCL, "%s failed: %s", #expr, nccl().GetErrorString(r_));      \
    } while (0)

#define HALO_GUARD_BEGIN try {
#define HALO_GUARD_END                                                                        \
    }                                                                                         \
    catch (const std::bad_alloc &) {                                                          \
        return fail(HALO_ENOMEM, "host allocation failed");                                  \
    }                                                                                         \
    catch (...) {                                                                             \
        return fail(HALO_EINVAL, "internal error");                                          \
    }

struct DeviceGuard {
    int prev = -1;
    bool active = false;
    explicit DeviceGuard(const halo_pool p) {
        if (p && !p->host_only) {
            cudaGetDevice(&prev);
            if (prev != p->cfg.device) {
                cudaSetDevice(p->cfg.device);
                active = true;
            }
        }
    }
    ~DeviceGuard() {
        if (active) cudaSetDevice(prev);
    }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

size_t storage_bytes(const halo_pool_config &c) {
    return (size_t)c.num_layers * (size_t)c.capacity_blocks * (size_t)c.num_kv_heads *
           (size_t)kBlockTok * (size_t)c.head_dim * 2;
}

bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// ---------------------------------------------------------------- NCCL (resolved at run time)
// The library does not link NCCL: it binds to the libnccl.so.2 already loaded in the
// process (torch's), or loads one on first use.  This keeps the .so loadable everywhere
// and avoids two NCCL versions in one process.
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommInitRankConfig)(ncclComm_t *, int, ncclUniqueId, int, ncclConfig_t *) = nullptr;
};

const NcclApi &nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
        a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
        a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
        a.Send = (decltype(a.Send))dlsym(h, "ncclSend");
        a.Recv = (decltype(a.Recv))dlsym(h, "ncclRecv");
        a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
        a.GroupStart = (decltype(a.GroupStart))dlsym(h, "ncclGroupStart");
        a.GroupEnd = (decltype(a.GroupEnd))dlsym(h, "ncclGroupEnd");
        a.CommInitRankConfig = (decltype(a.CommInitRankConfig))dlsym(h, "ncclCommInitRankConfig");
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv && a.GetErrorString &&
               a.GroupStart && a.GroupEnd;
        return a;
    }();
    return api;
}

// ---------------------------------------------------------------- block allocator
cudaEvent_t get_event(halo_pool p) {
    if (!p->event_cache.empty()) {
        cudaEvent_t e = p->event_cache.back();
        p->event_cache.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    return e;
}

void note_stream(halo_pool p, cudaStream_t s) {
    if (p->host_only) return;
    ++p->use_clock;
    for (auto &f : p->streams)
        if (f.stream == s) {
            f.last_use = p->use_clock;
            return;
        }
    if (p->streams.size() >= 16) {
        // forget the least recently used stream -- after its enqueued work has finished, so a
        // later release (which fences only the listed streams) cannot free blocks it still reads
        auto it = std::min_element(p->streams.begin(), p->streams.end(),
                                   [](const StreamFence &a, const StreamFence &b) {
                                       return a.last_use < b.last_use;
                                   });
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(it->stream, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone)
            cudaStreamSynchronize(it->stream);
        cudaGetLastError();
        *it = StreamFence{s, p->use_clock};
    } else {
        p->streams.push_back(StreamFence{s, p->use_clock});
    }
}

// A node fetched on another stream (background prefetch): order `s` after its copies.
halo_status wait_ready(halo_pool p, const Node &n, cudaStream_t s) {
    if (p->host_only || !n.ready) return HALO_OK;
    return cudaStreamWaitEvent(s, n.ready, 0) == cudaSuccess ? HALO_OK
                                                             : report_error(HALO_ECUDA, "cudaStreamWaitEvent failed");
}

void reclaim(halo_pool p, bool wait) {
    for (size_t i = 0; i < p->pending.size();) {
        PendingFree &pf = p->pending[i];
        bool done = true;
        for (cudaEvent_t e : pf.events) {
            cudaError_t r = wait ? cudaEventSynchronize(e) : cudaEventQuery(e);
            if (r == cudaErrorNotReady) {
                done = false;
                break;
            }
            if (r != cudaSuccess) cudaGetLastError();
        }
        if (!done) {
            ++i;
            continue;
        }
        for (auto it = pf.blocks.rbegin(); it != pf.blocks.rend(); ++it) p->free_list.push_back(*it);
        for (cudaEvent_t e : pf.events) p->event_cache.push_back(e);
        p->pending.erase(p->pending.begin() + i);
    }
}

halo_status alloc_blocks(halo_pool p, int64_t n, std::vector<int32_t> &out) {
    if ((int64_t)p->free_list.size() < n) reclaim(p, false);
    if ((int64_t)p->free_list.size() < n) reclaim(p, true);
    if ((int64_t)p->free_list.size() < n)
        return fail(HALO_ENOMEM, "pool out of blocks: need %lld, free %lld", (long long)n,
                    (long long)p->free_list.size());
    out.reserve(out.size() + n);
    ++p->epoch;  // a new owner: its V-table writes outrank every earlier owner's
    for (int64_t i = 0; i < n; ++i) {
        out.push_back(p->free_list.back());
        p->blk_epoch[out.back()] = p->epoch;
        p->free_list.pop_back();
    }
    return HALO_OK;
}

// Allocation epochs of the blocks of `slots` (token slots) or of `blocks`.
std::vector<uint32_t> slot_tags(halo_pool p, const std::vector<int32_t> &slots) {
    std::vector<uint32_t> t(slots.size());
    for (size_t i = 0; i < slots.size(); ++i) t[i] = p->blk_epoch[slots[i] / kBlockTok];
    return t;
}
std::vector<uint32_t> block_tags(halo_pool p, const std::vector<int32_t> &blocks) {
    std::vector<uint32_t> t(blocks.size());
    for (size_t i = 0; i < blocks.size(); ++i) t[i] = p->blk_epoch[blocks[i]];
    return t;
}

// Return blocks that were never handed to the device (error paths).
void unalloc_blocks(halo_pool p, const std::vector<int32_t> &blocks, size_t from) {
    for (size_t i = blocks.size(); i > from; --i) p->free_list.push_back(blocks[i - 1]);
}

// Blocks become reusable once the work enqueued so far on every stream that used the
// pool has passed (events recorded now).
void release_blocks(halo_pool p, std::vector<int32_t> &&blocks) {
    if (blocks.empty()) return;
    p->layout_gen++;  // plans built before this may read these blocks: they are stale now
    if (p->host_only) {
        for (auto it = blocks.rbegin(); it != blocks.rend(); ++it) p->free_list.push_back(*it);
        return;
    }
    PendingFree pf;
    pf.blocks = std::move(blocks);
    for (auto &f : p->streams) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(f.stream, &cs) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if (cs != cudaStreamCaptureStatusNone) continue;
        cudaEvent_t e = get_event(p);
        if (e && cudaEventRecord(e, f.stream) == cudaSuccess) pf.events.push_back(e);
        else cudaGetLastError();
    }
    p->pending.push_back(std::move(pf));
}

// ---------------------------------------------------------------- device scratch
struct Scratch {
    void *ptr = nullptr;
    cudaStream_t s = nullptr;
    ~Scratch() {
        if (ptr) cudaFreeAsync(ptr, s);
    }
};

halo_status upload(const void *host, size_t bytes, cudaStream_t s, Scratch &sc) {
    sc.s = s;
    HALO_CUDA(cudaMallocAsync(&sc.ptr, bytes ? bytes : 16, s));
    if (bytes) HALO_CUDA(cudaMemcpyAsync(sc.ptr, host, bytes, cudaMemcpyHostToDevice, s));
    return HALO_OK;
}

// Same through the pool's pinned ring (no host wait behind other streams' copies).
halo_status upload(halo_pool p, const void *host, size_t bytes, cudaStream_t s, Scratch &sc) {
    sc.s = s;
    HALO_CUDA(cudaMallocAsync(&sc.ptr, bytes ? bytes : 16, s));
    if (!bytes) return HALO_OK;
    void *h = p->pin_up.acquire(bytes);
    if (!h) return fail(HALO_ENOMEM, "pinned staging of %zu bytes", bytes);
    memcpy(h, host, bytes);
    HALO_CUDA(p->pin_up.commit(sc.ptr, bytes, s));
    return HALO_OK;
}

// Device copy of a host-or-device input.
halo_status as_device(const void *p, size_t bytes, cudaStream_t s, Scratch &sc, const void **out) {
    if (is_device_ptr(p)) {
        *out = p;
        return HALO_OK;
    }
    halo_status st = upload(p, bytes, s, sc);
    if (st != HALO_OK) return st;
    *out = sc.ptr;
    return HALO_OK;
}

halo_status check_pool(halo_pool p) {
    if (!p) return fail(HALO_EINVAL, "null pool");
    return HALO_OK;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

halo_status make_tmap(halo_pool p, void *base, CUtensorMap *out, int box_blocks) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *f = nullptr;
        HALO_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
        if (!f || q != cudaDriverEntryPointSuccess)
            return fail(HALO_ECUDA, "cuTensorMapEncodeTiled unavailable");
        fn = (EncodeTiledFn)f;
    }
    const auto &c = p->cfg;
    // dims (innermost first): d, token-in-block, kv head, layer*capacity + block
    cuuint64_t dims[4] = {(cuuint64_t)c.head_dim, (cuuint64_t)kBlockTok, (cuuint64_t)c.num_kv_heads,
                          (cuuint64_t)c.num_layers * (cuuint64_t)c.capacity_blocks};
    cuuint64_t strides[3] = {(cuuint64_t)c.head_dim * 2, (cuuint64_t)kBlockTok * c.head_dim * 2,
                             (cuuint64_t)c.num_kv_heads * kBlockTok * c.head_dim * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)kBlockTok, 1, (cuuint32_t)box_blocks};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(HALO_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return HALO_OK;
}

// K1's Q map: q bf16 [nreq][hq][d] as dims {d, hq, nreq}; box {64, g, 128/g} = one
// 128-row sub-tile (rows = request-major, q head of the kv group minor) per 64-wide d atom.
halo_status make_qmap(halo_pool p, const void *q, int32_t nreq, CUtensorMap *out) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult qr;
        void *f = nullptr;
        HALO_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr));
        if (!f || qr != cudaDriverEntryPointSuccess)
            return fail(HALO_ECUDA, "cuTensorMapEncodeTiled unavailable");
        fn = (EncodeTiledFn)f;
    }
    const auto &c = p->cfg;
    const int g = c.num_q_heads / c.num_kv_heads;
    cuuint64_t dims[3] = {(cuuint64_t)c.head_dim, (cuuint64_t)c.num_q_heads, (cuuint64_t)nreq};
    cuuint64_t strides[2] = {(cuuint64_t)c.head_dim * 2, (cuuint64_t)c.num_q_heads * c.head_dim * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)g, (cuuint32_t)(128 / g)};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(q), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(HALO_ECUDA, "cuTensorMapEncodeTiled (q) failed (%d)", (int)r);
    return HALO_OK;
}

// ---------------------------------------------------------------- plan builder
struct PNode {
    int64_t id;
    int parent;  // plan-local index or -1
    const Node *node;
    std::vector<int> children;
    int pre = 0, end = 0;  // preorder interval [pre, end)
    int r0 = 0, r1 = 0;    // request range in DFS order
    bool tensor = false;
    int splits = 0, chunk = 0;
    int slot_base = 0;
    int blk_off = 0;
};

// Choose a split-N chunk (tokens, multiple of 128) for the K1 nodes so the tiles fill the
// SMs: minimise an estimated makespan  max(longest tile, waves x mean tile)  where a tile
// costs its tokens plus a fixed per-tile overhead.
int choose_chunk(const std::vector<PNode> &ns, int g, int hkv, int nsm, int max_splits) {
    int64_t max_tok = 0;
    for (auto &n : ns)
        if (n.tensor) max_tok = std::max<int64_t>(max_tok, n.node->ntok);
    if (max_tok == 0) return kK1Tok;
    const int64_t kOvh = 256;
    const int64_t nk = ceil_div(std::min<int64_t>(max_tok, kK1MaxTileTok), kK1Tok);
    const int64_t step = std::max<int64_t>(1, nk / 256);
    double best = 1e300;
    int best_c = (int)(nk * kK1Tok);
    for (int64_t k = nk; k >= 1; k -= step) {
        const int64_t C = k * kK1Tok;
        int64_t T = 0;
        double sum = 0, maxc = 0;
        for (auto &n : ns) {
            if (!n.tensor) continue;
            const int64_t tok = n.node->ntok;
            int64_t s = std::max(std::min<int64_t>(ceil_div(tok, C), max_splits), ceil_div(tok, kK1MaxTileTok));
            const int64_t ch = ceil_div(ceil_div(tok, s), kK1Tok) * kK1Tok;
            s = ceil_div(tok, ch);
            const int64_t base = ceil_div((int64_t)(n.r1 - n.r0) * g, kK1Rows) * hkv;
            const double cost = (double)std::min(ch, tok) + kOvh;
            T += base * s;
            sum += (double)(base * s) * cost;
            maxc = std::max(maxc, cost);
        }
        const double est = std::max(maxc, (double)ceil_div(T, nsm) * (sum / (double)T));
        if (est < best * 0.999) {
            best = est;
            best_c = (int)C;
        }
    }
    return best_c;
}

// Plan options (halo_plan_options) with their defaults applied.
int k2_sms(halo_plan pl) {
    const int n = pl->opt.k2_sms, all = pl->pool->num_sms;
    return (n > 0 && n < all) ? n : all;
}
double k2_early_weight(halo_plan pl) { return pl->opt.k2_early_weight > 0 ? pl->opt.k2_early_weight : pl->k2_early_w; }
double k1_sm_frac(halo_plan pl) {
    const float f = pl->opt.k1_sm_frac;
    return f < 0 ? 0.0 : f == 0 ? 0.75 : (double)f;
}

// `virt` (prefill): the plan's rows are these virtual requests -- one per new prompt token,
// with its request's leaf and the prefix of its suffix blocks up to and including the token
// -- instead of the pool requests `reqs`.
// Prefill groups: the rows [first, first + ntok) of `virt` are the new tokens of one request
// whose suffix is `blocks` (len tokens); token t sees len - ntok + t + 1 suffix tokens.  When
// the group has enough rows for the tensor cores, its causal part runs as K1 tiles over the
// request's own blocks (and the rows' virtual suffixes are emptied for K2).
struct CausalGroup {
    int32_t first, ntok, len;
    const std::vector<int32_t> *blocks;
};

halo_status build_plan(halo_plan pl, int32_t nreq, const int64_t *reqs,
                       const std::vector<Request> *virt = nullptr,
                       const std::vector<CausalGroup> *causal = nullptr) {
    halo_pool p = pl->pool;
    const auto &cfg = p->cfg;
    const int g = cfg.num_q_heads / cfg.num_kv_heads;
    const int hkv = cfg.num_kv_heads, hq = cfg.num_q_heads, D = cfg.head_dim;
    const int min_rows = pl->opt.min_tensor_rows > 0 ? pl->opt.min_tensor_rows : 64;
    const int max_splits = pl->opt.max_splits > 0 ? pl->opt.max_splits : 16;

    // 1. requests
    std::vector<const Request *> R(nreq);
    for (int i = 0; i < nreq; ++i) {
        if (virt) {
            R[i] = &(*virt)[i];
            continue;
        }
        auto it = p->requests.find(reqs[i]);
        if (it == p->requests.end())
            return fail(HALO_ENOENT, "unknown request id %lld", (long long)reqs[i]);
        if (it->second.leaf < 0 && it->second.len == 0)
            return fail(HALO_EINVAL, "request %lld has an empty context", (long long)reqs[i]);
        R[i] = &it->second;
    }
    // 2. involved nodes
    std::vector<PNode> ns;
    std::unordered_map<int64_t, int> loc;
    std::vector<int> leaf_loc(nreq, -1);
    for (int i = 0; i < nreq; ++i) {
        int64_t id = R[i]->leaf;
        int child = -1;
        while (id >= 0) {
            auto f = loc.find(id);
            if (f != loc.end()) {
                if (child >= 0) ns[child].parent = f->second;
                if (leaf_loc[i] < 0) leaf_loc[i] = f->second;
                break;
            }
            auto nit = p->nodes.find(id);
            if (nit == p->nodes.end()) return fail(HALO_EINVAL, "dangling node %lld", (long long)id);
            if (nit->second.on_host)
                return fail(HALO_EBUSY, "node %lld is offloaded to host memory: fetch it first", (long long)id);
            PNode pn;
            pn.id = id;
            pn.parent = -1;
            pn.node = &nit->second;
            ns.push_back(pn);
            const int me = (int)ns.size() - 1;
            loc[id] = me;
            if (child >= 0) ns[child].parent = me;
            if (leaf_loc[i] < 0) leaf_loc[i] = me;
            child = me;
            id = nit->second.parent;
        }
    }
    // LRU clock: every node this plan reads is "used now"
    ++p->plan_tick;
    for (auto &n : ns) const_cast<Node *>(n.node)->last_use = p->plan_tick;
    pl->layout_gen = p->layout_gen;
    // deterministic child order: by node id
    std::vector<int> roots;
    {
        std::vector<int> by_id(ns.size());
        for (size_t i = 0; i < ns.size(); ++i) by_id[i] = (int)i;
        std::sort(by_id.begin(), by_id.end(), [&](int a, int b) { return ns[a].id < ns[b].id; });
        for (int i : by_id) {
            if (ns[i].parent < 0) roots.push_back(i);
            else ns[ns[i].parent].children.push_back(i);
        }
    }
    // 3. DFS preorder
    std::vector<int> pre_order;
    {
        std::vector<std::pair<int, int>> st;  // (node, next child)
        for (int r : roots) {
            st.push_back({r, 0});
            ns[r].pre = (int)pre_order.size();
            pre_order.push_back(r);
            while (!st.empty()) {
                auto &top = st.back();
                PNode &n = ns[top.first];
                if (top.second < (int)n.children.size()) {
                    const int c = n.children[top.second++];
                    ns[c].pre = (int)pre_order.size();
                    pre_order.push_back(c);
                    st.push_back({c, 0});
                } else {
                    n.end = (int)pre_order.size();
                    st.pop_back();
                }
            }
        }
    }
    // 4. requests in DFS order of their leaves (no-prefix requests last)
    std::vector<int> key(nreq);
    for (int i = 0; i < nreq; ++i) key[i] = leaf_loc[i] >= 0 ? ns[leaf_loc[i]].pre : INT32_MAX;
    pl->req_order.resize(nreq);
    for (int i = 0; i < nreq; ++i) pl->req_order[i] = i;
    std::stable_sort(pl->req_order.begin(), pl->req_order.end(),
                     [&](int a, int b) { return key[a] < key[b]; });
    std::vector<int> sorted_keys(nreq);
    for (int i = 0; i < nreq; ++i) sorted_keys[i] = key[pl->req_order[i]];
    // 5./6. node request ranges and the K1 decision
    int tensor_nodes = 0;
    for (auto &n : ns) {
        n.r0 = (int)(std::lower_bound(sorted_keys.begin(), sorted_keys.end(), n.pre) - sorted_keys.begin());
        n.r1 = (int)(std::lower_bound(sorted_keys.begin(), sorted_keys.end(), n.end) - sorted_keys.begin());
        n.tensor = (int64_t)(n.r1 - n.r0) * g >= min_rows;
        tensor_nodes += n.tensor;
    }
    // 7. splits
    if (pl->opt.force_splits > 0) {
        for (auto &n : ns) {
            if (!n.tensor) continue;
            const int64_t tok = n.node->ntok;
            const int64_t s = std::max(std::min<int64_t>(pl->opt.force_splits, ceil_div(tok, kK1Tok)),
                                       ceil_div(tok, kK1MaxTileTok));
            n.chunk = (int)(ceil_div(ceil_div(tok, s), kK1Tok) * kK1Tok);
            n.splits = (int)ceil_div(tok, n.chunk);
        }
    } else {
        int C = choose_chunk(ns, g, hkv, p->num_sms, max_splits);
        // K1 in a single partial wave beside a K2 that dominates the layer (co-schedule model).
        // Under programmatic dependent launch K2's first (SMs - K1 CTAs) CTAs stream on the SMs
        // K1 leaves idle; K2 parks finished units until K1 is done.  For each split count whose
        // tiles fit one wave the model estimates
        //   T1 = t0 + t_n * (n-tiles per K1 CTA)                  (K1 CTA duration)
        //   early = E * r_e * T1                                  (E = SMs - K1 CTAs)
        //   T  = T1 + max(0, B - early) / R                       (B = K2 bytes, R = HBM)
        // and takes the split count of least T (if it beats the default tiling).  K2's early CTAs
        // get w = (r_e T1 + r_pe T2) / (r_pl T2) times a late CTA's share (T2 = T - T1; CTAs
        // already streaming keep more of the bandwidth after K1 than the ones entering then).
        // Constants measured on B200 (round 2: tools/k1k2_cosched_sweep.py, tools/k2_trace.py,
        // profiles/k1k2_cosched_r02b.txt, k2_trace_cosched_r02.txt); r_pe and r_pl re-measured
        // on the session-3 K2 (cheaper unit ends): PDL trace at w = 3.0, balanced (early / late
        // CTAs exit at 55.6 / 54.8 us): late CTAs 0.90 MB in 30.5 us = 29 GB/s, early CTAs
        // 2.69 MB = 44 x 24.3 + r_pe x 31.3 -> 52 GB/s (profiles/k2_trace_w3_r02.txt).
        pl->k2_early = false;
        pl->k2_early_w = 1.0;
        if (k1_sm_frac(pl) > 0 && pl->opt.max_splits <= 0) {
            constexpr double kT0 = 3.0, kTn = 2.75;          // us: K1 CTA prologue+epilogue, per n-tile
            constexpr double kRe = 44e3, kRpe = 52e3, kRpl = 29e3;  // bytes/us per SM: beside K1, after K1
            constexpr double kR = 6.2e6;                     // bytes/us: HBM, K2 streaming on all SMs
            auto tiles_for = [&](int64_t Cc, int64_t &max_ch) {
                int64_t T = 0;
                max_ch = 0;
                for (auto &n : ns) {
                    if (!n.tensor) continue;
                    const int64_t tok = n.node->ntok;
                    int64_t sp = std::max(std::min<int64_t>(ceil_div(tok, Cc), max_splits), ceil_div(tok, kK1MaxTileTok));
                    const int64_t ch = ceil_div(ceil_div(tok, sp), kK1Tok) * kK1Tok;
                    sp = ceil_div(tok, ch);
                    T += ceil_div((int64_t)(n.r1 - n.r0) * g, kK1Rows) * hkv * sp;
                    max_ch = std::max(max_ch, std::min(ch, tok));
                }
                return T;
            };
            double B = 0;
            for (int i = 0; i < nreq; ++i) B += (double)R[i]->blocks.size() * kBlockTok * hkv * D * 4;
            const int sms = k2_sms(pl);
            auto model = [&](int64_t tiles, int64_t max_ch, double &w) {
                const double t1 = kT0 + kTn * (double)ceil_div(max_ch, kK1Tok);
                const int64_t waves = ceil_div(tiles, (int64_t)sms);
                if (waves > 1) {  // multi-wave K1: K2 streams beside its last wave only (ignored)
                    w = 1.0;
                    return (double)waves * t1 + B / kR;
                }
                const double E = (double)(sms - tiles), re = std::min(kRe, kR / std::max(E, 1.0));
                const double rest = std::max(0.0, B - E * re * t1);
                const double t2 = rest / kR;
                w = t2 > 0 ? std::min(8.0, std::max(1.0, (re * t1 + kRpe * t2) / (kRpl * t2))) : 8.0;
                return t1 + t2;
            };
            int64_t mc = 0;
            double w0 = 1.0;
            const int64_t tiles0 = tiles_for(C, mc);  // (sets mc: not inside the call's arguments)
            const double base = model(tiles0, mc, w0);
            double best = base * 0.98;  // switch only for a clear gain
            // only when K2 dominates the layer: its HBM time >= 1.25x the default K1 CTA time,
            // and >= 8 blocks per K2 warp (with fewer, K2 is bound by per-unit latency, which the
            // model does not capture: 64 x 8192-token fan-out lost 13% with the rule)
            const double t1_base = kT0 + kTn * (double)ceil_div(mc, kK1Tok);
            const double blocks_per_warp = B / ((double)kBlockTok * hkv * D * 4) * hkv / ((double)sms * kK2WarpsWide);
            if (B / kR < 1.25 * t1_base || blocks_per_warp < 8.0) best = 0;
            for (int64_t Cc = kK1Tok; Cc <= kK1MaxTileTok && best > 0; Cc += kK1Tok) {
                const int64_t T1 = tiles_for(Cc, mc);
                // K1 on 40..k1_sm_frac of the SMs: with fewer K1 CTAs (longer tiles) the measured
                // layer time departs from the model (C1, 32 CTAs: 75 us measured vs 54 modeled)
                if (T1 <= 0 || T1 > (int64_t)(k1_sm_frac(pl) * sms) || T1 >= sms || T1 < (int64_t)(0.4 * sms))
                    continue;
                double w = 1.0;
                const double t = model(T1, mc, w);
                if (t < best) {
                    best = t;
                    C = (int)Cc;
                    pl->k2_early = true;
                    pl->k2_early_w = w;
                }
            }
        }
        for (auto &n : ns) {
            if (!n.tensor) continue;
            const int64_t tok = n.node->ntok;
            const int64_t s = std::max(std::min<int64_t>(ceil_div(tok, C), max_splits), ceil_div(tok, kK1MaxTileTok));
            n.chunk = (int)(ceil_div(ceil_div(tok, s), kK1Tok) * kK1Tok);
            n.splits = (int)ceil_div(tok, n.chunk);
        }
    }
    // 8. slot bases along each path (preorder visits parents first)
    for (int i : pre_order) {
        PNode &n = ns[i];
        n.slot_base = n.parent < 0 ? 0
                                   : ns[n.parent].slot_base + (ns[n.parent].tensor ? ns[n.parent].splits : 0);
    }
    pl->req_nslots.assign(nreq, 0);
    int max_slots = 0;
    for (int i = 0; i < nreq; ++i) {
        if (leaf_loc[i] >= 0) {
            const PNode &lf = ns[leaf_loc[i]];
            pl->req_nslots[i] = lf.slot_base + (lf.tensor ? lf.splits : 0);
        }
        max_slots = std::max(max_slots, pl->req_nslots[i]);
    }
    // causal K1 groups (prefill): one more partial slot for each of their rows
    std::vector<char> causal_k1(causal ? causal->size() : 0, 0);
    if (causal) {
        for (size_t c = 0; c < causal->size(); ++c) {
            const CausalGroup &cg = (*causal)[c];
            if ((int64_t)cg.ntok * g < min_rows || cg.len > kK1MaxTileTok) continue;
            causal_k1[c] = 1;
            for (int32_t t = 0; t < cg.ntok; ++t) {
                const int i = cg.first + t;
                pl->req_nslots[i] += 1;
                max_slots = std::max(max_slots, pl->req_nslots[i]);
            }
        }
    }
    // 9./10. K1 node blocks and tiles
    pl->node_blocks.clear();
    pl->tiles.clear();
    std::vector<int32_t> tile_causal;  // per tile: visible-token offset of its first row, or -1
    double k1_flops = 0, k1_bytes = 0;
    for (int i : pre_order) {
        PNode &n = ns[i];
        if (!n.tensor) continue;
        n.blk_off = (int)pl->node_blocks.size();
        pl->node_blocks.insert(pl->node_blocks.end(), n.node->blocks.begin(), n.node->blocks.end());
        const int64_t rows = (int64_t)(n.r1 - n.r0) * g;
        const int64_t tok = n.node->ntok;
        k1_flops += 4.0 * rows * tok * D * hkv;
        k1_bytes += (double)tok * hkv * D * 2 * 2 + (double)rows * hkv * D * 2 +
                    (double)rows * hkv * (D + 1) * 4 * n.splits;
        for (int64_t m0 = 0; m0 < rows; m0 += kK1Rows)
            for (int j = 0; j < hkv; ++j)
                for (int s = 0; s < n.splits; ++s) {
                    PrefixTile t;
                    t.req_off = n.r0 + (int32_t)(m0 / g);
                    t.nrows = (int32_t)std::min<int64_t>(kK1Rows, rows - m0);
                    t.kv_head = j;
                    t.tok_begin = s * n.chunk;
                    t.tok_end = (int32_t)std::min<int64_t>(tok, (int64_t)(s + 1) * n.chunk);
                    t.blk_off = n.blk_off;
                    t.slot = n.slot_base + s;
                    t.node = i;
                    pl->tiles.push_back(t);
                    tile_causal.push_back(-1);
                }
    }
    if (causal) {
        // DFS position of every row (caller index -> position in req_order)
        std::vector<int32_t> pos(nreq);
        for (int r = 0; r < nreq; ++r) pos[pl->req_order[r]] = r;
        for (size_t c = 0; c < causal->size(); ++c) {
            if (!causal_k1[c]) continue;
            const CausalGroup &cg = (*causal)[c];
            const int32_t blk_off = (int32_t)pl->node_blocks.size();
            pl->node_blocks.insert(pl->node_blocks.end(), cg.blocks->begin(), cg.blocks->end());
            const int64_t rows = (int64_t)cg.ntok * g;
            const int32_t base = cg.len - cg.ntok;  // suffix tokens before the prompt
            for (int32_t t = 0; t < cg.ntok; ++t)
                k1_flops += 4.0 * g * (base + t + 1) * D * hkv;
            k1_bytes += (double)cg.len * hkv * D * 4 + (double)rows * hkv * D * 2 + (double)rows * hkv * (D + 1) * 4;
            for (int64_t m0 = 0; m0 < rows; m0 += kK1Rows)
                for (int j = 0; j < hkv; ++j) {
                    PrefixTile t;
                    t.req_off = pos[cg.first] + (int32_t)(m0 / g);
                    t.nrows = (int32_t)std::min<int64_t>(kK1Rows, rows - m0);
                    t.kv_head = j;
                    t.tok_begin = 0;
                    // the tile's last row sees base + (m0 + nrows)/g tokens: nothing after
                    t.tok_end = std::min<int32_t>(cg.len, base + (int32_t)((m0 + t.nrows + g - 1) / g));
                    t.blk_off = blk_off;
                    t.slot = pl->req_nslots[cg.first] - 1;
                    t.node = -1;
                    pl->tiles.push_back(t);
                    tile_causal.push_back(base + (int32_t)(m0 / g));
                }
        }
    }
    {
        std::vector<size_t> idx(pl->tiles.size());
        for (size_t k = 0; k < idx.size(); ++k) idx[k] = k;
        std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
            return (pl->tiles[a].tok_end - pl->tiles[a].tok_begin) > (pl->tiles[b].tok_end - pl->tiles[b].tok_begin);
        });
        std::vector<PrefixTile> t2(idx.size());
        std::vector<int32_t> c2(idx.size());
        for (size_t k = 0; k < idx.size(); ++k) {
            t2[k] = pl->tiles[idx[k]];
            c2[k] = tile_causal[idx[k]];
        }
        pl->tiles.swap(t2);
        tile_causal.swap(c2);
    }
    // 10b. per-tile shortcuts that save K1 a dependent global load each: the caller index of
    // the tile's first request when its requests are consecutive caller indices (q rows are
    // then addressed directly), and the pool block of its first token when the node's blocks
    // over the tile's range are physically consecutive (TMA coordinates computed, no block list)
    pl->tile_aux.assign(pl->tiles.size() * 4, -1);
    for (size_t ti = 0; ti < pl->tiles.size(); ++ti) {
        const PrefixTile &t = pl->tiles[ti];
        const int nr = (t.nrows + g - 1) / g;
        bool rc = true;
        for (int i = 1; i < nr && rc; ++i) rc = pl->req_order[t.req_off + i] == pl->req_order[t.req_off] + i;
        if (rc) pl->tile_aux[4 * ti] = pl->req_order[t.req_off];
        const int b0 = t.tok_begin / kBlockTok, b1 = (t.tok_end + kBlockTok - 1) / kBlockTok;
        bool bc = true;
        for (int b = b0 + 1; b < b1 && bc; ++b) bc = pl->node_blocks[t.blk_off + b] == pl->node_blocks[t.blk_off + b - 1] + 1;
        if (bc) pl->tile_aux[4 * ti + 1] = pl->node_blocks[t.blk_off + b0];
        if (tile_causal[ti] >= 0) {  // causal prefill tile: row r sees w + r/g + 1 tokens
            pl->tile_aux[4 * ti + 2] = 1;
            pl->tile_aux[4 * ti + 3] = tile_causal[ti];
        }
    }
    // rows whose causal part runs in K1 stream no suffix blocks in K2
    std::vector<char> skip_suffix(nreq, 0);
    if (causal)
        for (size_t c = 0; c < causal->size(); ++c)
            if (causal_k1[c])
                for (int32_t t = 0; t < (*causal)[c].ntok; ++t) skip_suffix[(*causal)[c].first + t] = 1;
    // 11. K2 per-request block lists: folded path nodes root -> leaf, then the suffix
    pl->req_blk_off.assign(nreq + 1, 0);
    pl->req_blk.clear();
    double k2_bytes = 0, unshared = 0;
    std::vector<int> path;
    auto push_blocks = [&](const std::vector<int32_t> &blocks, int32_t ntok) {
        for (size_t b = 0; b < blocks.size(); ++b) {
            const int32_t cnt = std::min<int32_t>(kBlockTok, ntok - (int32_t)b * kBlockTok);
            pl->req_blk.push_back((uint32_t)blocks[b] | ((uint32_t)(cnt - 1) << kBlkCountShift));
        }
    };
    int folded = 0;
    for (auto &n : ns) folded += !n.tensor;
    std::vector<int32_t> req_fold_blk(nreq, 0);  // leading blocks of folded (shared) path nodes
    for (int i = 0; i < nreq; ++i) {
        pl->req_blk_off[i] = (int32_t)pl->req_blk.size();
        const size_t fold0 = pl->req_blk.size();
        path.clear();
        for (int x = leaf_loc[i]; x >= 0; x = ns[x].parent) path.push_back(x);
        int64_t ctx = R[i]->len;
        for (auto it = path.rbegin(); it != path.rend(); ++it) {
            const PNode &n = ns[*it];
            ctx += n.node->ntok;
            if (!n.tensor) push_blocks(n.node->blocks, n.node->ntok);
        }
        req_fold_blk[i] = (int32_t)(pl->req_blk.size() - fold0);
        if (!skip_suffix[i]) push_blocks(R[i]->blocks, R[i]->len);
        unshared += (double)ctx * hkv * D * 4;
    }
    pl->req_blk_off[nreq] = (int32_t)pl->req_blk.size();
    k2_bytes = (double)pl->req_blk.size() * kBlockTok * hkv * D * 4 + (double)nreq * hq * D * 2 +
               (double)nreq * hq * (D + 1) * 4;
    for (int i = 0; i < nreq; ++i) k2_bytes += (double)pl->req_nslots[i] * hq * (D + 1) * 4;
    if (pl->req_blk.empty()) k2_bytes -= (double)nreq * hq * D * 2;  // K3 alone reads no q
    // 12. K2 request order: longest block list first (LPT), stable
    pl->unit_req.resize(nreq);
    for (int i = 0; i < nreq; ++i) pl->unit_req[i] = i;
    std::stable_sort(pl->unit_req.begin(), pl->unit_req.end(), [&](int a, int b) {
        return pl->req_blk_off[a + 1] - pl->req_blk_off[a] > pl->req_blk_off[b + 1] - pl->req_blk_off[b];
    });
    // 12b. K2 schedule: static chunks, warp w takes chunks w, w + W, ...
    // Work items: unit u = its n_u blocks followed by one merge item (the K3 epilogue), so
    // units with few or no blocks (prefill rows whose causal part ran in K1) still spread
    // over the warps.  Chunks are contiguous item ranges of about equal weight.
    {
        const int U = nreq * hkv;
        const int64_t Ww = (int64_t)k2_sms(pl) * kK2WarpsWide, Wn = (int64_t)k2_sms(pl) * kK2WarpsNarrow;
        pl->k2_warps = kK2WarpsWide;
        pl->unit_boff.assign(U + 1, 0);
        for (int u = 0; u < U; ++u) {
            const int req = pl->unit_req[u / hkv];
            pl->unit_boff[u + 1] = pl->unit_boff[u] + (pl->req_blk_off[req + 1] - pl->req_blk_off[req]);
        }
        const int64_t Btot = pl->unit_boff[U], Itot = Btot + U;
        auto ui = [&](int64_t u) { return (int64_t)pl->unit_boff[u] + u; };  // items before unit u
        auto nb = [&](int64_t u) { return (int64_t)pl->unit_boff[u + 1] - pl->unit_boff[u]; };
        // item -> unit map (O(1) lookups: the cut computations below do thousands of them)
        std::vector<int32_t> &umap = pl->item_unit;
        umap.resize((size_t)Itot);
        for (int u = 0; u < U; ++u)
            std::fill(umap.begin() + ui(u), umap.begin() + ui(u + 1), (int32_t)u);
        auto unit_of = [&](int64_t x) -> int64_t {  // unit owning item x < Itot
            return umap[(size_t)std::min(std::max<int64_t>(x, 0), Itot - 1)];
        };
        // a cut never separates a unit's merge item from its last block (that chunk would
        // visit the unit with no blocks)
        auto push_cut = [&](std::vector<int64_t> &c, int64_t x) {
            if (x > 0 && x < Itot) {
                const int64_t u = unit_of(x);
                if (nb(u) > 0 && x - ui(u) == nb(u)) ++x;
            }
            if (x > c.back() && x < Itot) c.push_back(x);
        };
        // Under programmatic dependent launch K2's CTAs are dispatched in blockIdx order: the
        // first num_sms - (K1 CTAs) land on SMs K1 leaves idle and stream while K1 runs; the
        // rest enter as K1's CTAs retire.  Warps of the early CTAs get `ew` times the share.
        const int64_t k1c = (int64_t)pl->tiles.size();
        const int64_t early_ctas = (k1c > 0 && k1c < k2_sms(pl)) ? k2_sms(pl) - k1c : 0;
        double ew = early_ctas > 0 && (pl->k2_early || pl->opt.k2_early_weight > 0) ? k2_early_weight(pl) : 1.0;
        auto target = [&](int64_t w, int64_t nw, int wpc) -> int64_t {  // item position of cut w
            if (ew == 1.0) return w * Itot / nw;
            const int64_t ne = std::min<int64_t>(nw, early_ctas * wpc);
            const double tot = (double)ne * ew + (double)(nw - ne);
            const double cw = (double)std::min<int64_t>(w, ne) * ew + (double)std::max<int64_t>(0, w - ne);
            return (int64_t)(cw / tot * (double)Itot);
        };
        auto equal_cuts = [&](int64_t nw, int wpc) {
            std::vector<int64_t> c(1, 0);
            for (int64_t w = 1; w < nw; ++w) push_cut(c, target(w, nw, wpc));
            c.push_back(Itot);
            return c;
        };
        // cuts snapped to the nearest unit boundary; `balanced` if the largest chunk stays
        // within 5% of the equal share (whole units: no stream-K merges)
        auto snapped_cuts = [&](int64_t nw, int wpc, bool &balanced) {
            std::vector<int64_t> c(1, 0);
            for (int64_t w = 1; w < nw && Itot > 0; ++w) {
                const int64_t x = target(w, nw, wpc), u = unit_of(x);
                const int64_t y = (x - ui(u) <= ui(u + 1) - x) ? ui(u) : ui(u + 1);
                if (y > c.back() && y < Itot) c.push_back(y);
            }
            c.push_back(Itot);
            // largest chunk against its warp's (weighted) share
            balanced = true;
            for (size_t k = 1; k < c.size(); ++k) {
                const int64_t w = (int64_t)k - 1;
                const int64_t share = std::max<int64_t>(1, ceil_div(target(w + 1, nw, wpc) - target(w, nw, wpc), 1));
                if ((c[k] - c[k - 1]) * 100 > std::max<int64_t>(share, ceil_div(Itot, nw)) * 105) balanced = false;
            }
            return c;
        };
        std::vector<int64_t> cuts;
        bool bal = false;
        // 1-3 whole units per narrow warp (halo_plan_options.k2_whole_units < 0: off)
        const bool few_units = pl->opt.k2_whole_units >= 0 && U > Ww && U <= 3 * Wn;
        if (pl->opt.k2_chunk_blocks > 0) {  // fixed-size chunks (tests)
            cuts.assign(1, 0);
            for (int64_t x = pl->opt.k2_chunk_blocks; x < Itot; x += pl->opt.k2_chunk_blocks) push_cut(cuts, x);
            cuts.push_back(Itot);
        } else if (pl->opt.k2_shape == 2) {  // forced narrow shape
            pl->k2_warps = kK2WarpsNarrow;
            cuts = equal_cuts(Wn, kK2WarpsNarrow);
        } else if (pl->opt.k2_shape == 1) {  // forced wide shape
            cuts = equal_cuts(Ww, kK2WarpsWide);
        } else if (((Btot < 8 * (int64_t)U && U < 2 * Ww) || (k1c == 0 && few_units)) &&
                   (cuts = snapped_cuts(Wn, kK2WarpsNarrow, bal), bal)) {
            // few units per warp (stream-K pieces would dominate: C1 has 1.15 units per wide
            // warp, so nearly every unit would be cut in two, and each merge costs the piece
            // that finishes last several memory round trips at the end of the kernel) and whole
            // units divide evenly over the narrow shape: 7 warps x 4 stages per SM, no pieces.
            // Only without K1 in the plan: beside K1 (under PDL) the wide shape with pieces
            // measured faster (C1: 53.6 vs 59.9 us per layer, profiles/k2_narrow_r02.txt);
            // such plans get the whole-unit schedule for K2 launched alone (below).
            pl->k2_warps = kK2WarpsNarrow;
        } else {
            cuts = snapped_cuts(Ww, kK2WarpsWide, bal);
            if (!bal) cuts = equal_cuts(Ww, kK2WarpsWide);  // equal item ranges (stream-K pieces)
        }
        if (cuts.size() < 2) cuts = {0, Itot};
        // static-then-dynamic: the wide shape's stream-K cuts get a dynamic tail -- the warps'
        // static shares cover the first (100 - tail)% of the items, the rest is cut into
        // pieces of about `piece` items that warps claim once their share is done
        pl->dyn_first = (int32_t)cuts.size() - 1;
        {
            const int tail_pct = std::max(0, pl->opt.k2_tail_pct);  // off by default (A/B: tools/k2_tail_ab.sh)
            const int64_t W = (int64_t)k2_sms(pl) * pl->k2_warps;
            const bool eligible = tail_pct > 0 && pl->opt.k2_chunk_blocks <= 0 && pl->k2_warps == kK2WarpsWide &&
                                  !bal && Itot >= 8 * W;
            if (eligible) {
                const int64_t front = Itot - Itot * std::min(tail_pct, 50) / 100;
                std::vector<int64_t> c(1, 0);
                for (int64_t w = 1; w < W; ++w) push_cut(c, target(w, W, pl->k2_warps) * front / Itot);
                push_cut(c, front);
                if ((int64_t)c.size() - 1 == W) {  // exactly one static chunk per warp
                    const int64_t piece = std::max<int64_t>(2, (Itot - front) / (2 * W));
                    for (int64_t x = front + piece; x < Itot; x += piece) push_cut(c, x);
                    c.push_back(Itot);
                    cuts.swap(c);
                    pl->dyn_first = (int32_t)W;
                }
            }
        }
        const int64_t nchunks = (int64_t)cuts.size() - 1;
        if (pl->dyn_first > nchunks) pl->dyn_first = (int32_t)nchunks;
        auto block_at = [&](int64_t x) {  // global block index where item x starts
            if (x >= Itot) return Btot;
            const int64_t u = unit_of(x);
            return (int64_t)pl->unit_boff[u] + std::min(x - ui(u), nb(u));
        };
        std::vector<int32_t> &lo = pl->chunk_lo;
        lo.resize(nchunks + 1);
        for (int64_t c = 0; c <= nchunks; ++c) lo[c] = (int32_t)block_at(cuts[c]);
        std::vector<int32_t> &cmap = pl->item_chunk;  // item -> chunk
        auto fill_cmap = [&](const std::vector<int64_t> &c) {
            cmap.resize((size_t)Itot);
            for (size_t k = 0; k + 1 < c.size(); ++k)
                std::fill(cmap.begin() + c[k], cmap.begin() + std::min(c[k + 1], Itot), (int32_t)k);
        };
        fill_cmap(cuts);
        auto chunk_of = [&](int64_t x) -> int64_t { return cmap[(size_t)x]; };
        pl->chunk_u0.assign(nchunks, 0);
        pl->chunk_u1.assign(nchunks, 0);
        for (int64_t c = 0; c < nchunks && U > 0; ++c) {
            if (cuts[c + 1] <= cuts[c]) continue;
            pl->chunk_u0[c] = (int32_t)unit_of(cuts[c]);
            pl->chunk_u1[c] = (int32_t)unit_of(cuts[c + 1] - 1) + 1;
        }
        pl->unit_nseg.resize(U);
        pl->unit_seg.resize(U);
        pl->unit_chunk0.resize(U);
        int32_t nseg_total = 0;
        for (int uu = 0; uu < U; ++uu) {
            const int64_t c0 = chunk_of(ui(uu)), c1 = chunk_of(ui(uu + 1) - 1);
            const int nseg = (int)(c1 - c0 + 1);
            pl->unit_chunk0[uu] = (int32_t)c0;
            pl->unit_nseg[uu] = nseg;
            pl->unit_seg[uu] = nseg > 1 ? nseg_total : -1;
            if (nseg > 1) nseg_total += nseg;
        }
        pl->nseg_total = nseg_total;
        pl->chunk_info.resize((size_t)nchunks * 4);
        for (int64_t cc = 0; cc < nchunks; ++cc) {
            pl->chunk_info[4 * cc] = lo[cc];
            pl->chunk_info[4 * cc + 1] = lo[cc + 1];
            pl->chunk_info[4 * cc + 2] = pl->chunk_u0[cc];
            pl->chunk_info[4 * cc + 3] = pl->chunk_u1[cc];
        }
        // per-block descriptors and per-unit metadata read by the kernel
        pl->k2_ent.resize((size_t)Btot * 2);
        pl->unit_meta.resize((size_t)U * 8);
        for (int uu = 0; uu < U; ++uu) {
            const int req = pl->unit_req[uu / hkv], head = uu % hkv;
            const int32_t b0 = pl->unit_boff[uu], b1 = pl->unit_boff[uu + 1];
            const int32_t rb = pl->req_blk_off[req];
            for (int32_t x = b0; x < b1; ++x) {
                const int32_t j = x - b0;
                const uint32_t e = pl->req_blk[rb + j];
                const uint32_t slab = (e & kBlkMask) * (uint32_t)hkv + (uint32_t)head;
                pl->k2_ent[2 * (size_t)x] = slab | (e & ~kBlkMask) | (x == b0 ? 0x80000000u : 0u);
                // bit 31: a block of a folded prefix node, read by every request under the node:
                // K2 streams it with the default L2 policy instead of evict_first
                pl->k2_ent[2 * (size_t)x + 1] = (uint32_t)(req * hkv + head) |
                                                (j < req_fold_blk[req] ? 0x80000000u : 0u);
            }
            int32_t *um = &pl->unit_meta[(size_t)uu * 8];
            um[0] = b0; um[1] = b1; um[2] = req; um[3] = head;
            um[4] = pl->req_nslots[req]; um[5] = pl->unit_nseg[uu]; um[6] = pl->unit_seg[uu];
            um[7] = pl->unit_chunk0[uu];
        }
        // K2 launched ALONE (K1 complete before it starts: halo_decode_run_stages with only the
        // K2 bit) runs without the co-schedule's early-CTA weights: an equal-share schedule
        pl->alt_nchunks = 0;
        pl->alt_nseg_total = 0;
        pl->alt_k2_warps = pl->k2_warps;
        if (ew != 1.0 && pl->dyn_first == (int32_t)nchunks) {
            ew = 1.0;
            bool bal2 = false;
            // alone, a few whole units per warp over the narrow shape beat stream-K pieces
            // (C1 K2: 0.83 vs 0.75 of HBM, no merges at the kernel's end)
            std::vector<int64_t> ce;
            if (few_units && pl->opt.k2_shape == 0 && pl->opt.k2_chunk_blocks <= 0 &&
                (ce = snapped_cuts(Wn, kK2WarpsNarrow, bal2), bal2)) {
                pl->alt_k2_warps = kK2WarpsNarrow;
            } else {
                const int64_t Wk = (int64_t)k2_sms(pl) * pl->k2_warps;
                ce = snapped_cuts(Wk, pl->k2_warps, bal2);
                if (!bal2) ce = equal_cuts(Wk, pl->k2_warps);
            }
            if (ce.size() < 2) ce = {0, Itot};
            const int64_t ne = (int64_t)ce.size() - 1;
            fill_cmap(ce);
            auto chunk_of_e = [&](int64_t x) -> int64_t { return cmap[(size_t)x]; };
            pl->alt_chunk_info.assign((size_t)ne * 4, 0);
            for (int64_t c = 0; c < ne; ++c) {
                pl->alt_chunk_info[4 * c] = (int32_t)block_at(ce[c]);
                pl->alt_chunk_info[4 * c + 1] = (int32_t)block_at(ce[c + 1]);
                if (ce[c + 1] > ce[c] && U > 0) {
                    pl->alt_chunk_info[4 * c + 2] = (int32_t)unit_of(ce[c]);
                    pl->alt_chunk_info[4 * c + 3] = (int32_t)unit_of(ce[c + 1] - 1) + 1;
                }
            }
            pl->alt_unit_meta = pl->unit_meta;
            int32_t nst = 0;
            for (int uu = 0; uu < U; ++uu) {
                const int64_t c0 = chunk_of_e(ui(uu)), c1 = chunk_of_e(ui(uu + 1) - 1);
                const int nseg = (int)(c1 - c0 + 1);
                int32_t *um = &pl->alt_unit_meta[(size_t)uu * 8];
                um[5] = nseg;
                um[6] = nseg > 1 ? nst : -1;
                um[7] = (int32_t)c0;
                if (nseg > 1) nst += nseg;
            }
            pl->alt_nseg_total = nst;
            pl->alt_nchunks = (int32_t)ne;
        }
    }
    pl->waits.clear();
    for (auto &n : ns)
        if (n.node->ready) pl->waits.push_back(n.node->ready);
    // 13. info
    halo_plan_info &inf = pl->info;
    inf = halo_plan_info{};
    inf.nreq = nreq;
    inf.num_q_heads = hq;
    inf.num_kv_heads = hkv;
    inf.head_dim = D;
    inf.tensor_nodes = tensor_nodes;
    inf.folded_nodes = folded;
    inf.k1_tiles = (int32_t)pl->tiles.size();
    inf.k2_units = nreq * hkv;
    inf.max_slots = max_slots;
    inf.k2_warps = pl->k2_warps;
    inf.k1_flops = k1_flops;
    inf.k1_bytes = k1_bytes;
    inf.k2_bytes = k2_bytes;
    inf.unshared_bytes = unshared;
    pl->nreq = nreq;
    return HALO_OK;
}

size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

halo_status upload_plan(halo_plan pl, cudaStream_t s) {
    halo_pool p = pl->pool;
    // nodes fetched from the host arena on another stream (background prefetch): the plan's
    // stream waits for their copies (free once they have passed)
    if (!p->host_only)
        for (cudaEvent_t e : pl->waits) HALO_CUDA(cudaStreamWaitEvent(s, e, 0));
    const int nreq = pl->nreq;
    size_t off = 0;
    const size_t o_tiles = off; off = align16(off + pl->tiles.size() * sizeof(PrefixTile));
    const size_t o_order = off; off = align16(off + nreq * 4);
    const size_t o_nblk = off; off = align16(off + pl->node_blocks.size() * 4);
    const size_t o_unit = off; off = align16(off + nreq * 4);
    const size_t o_boff = off; off = align16(off + (nreq + 1) * 4);
    const size_t o_blk = off; off = align16(off + pl->req_blk.size() * 4);
    const size_t o_nsl = off; off = align16(off + nreq * 4);
    const int U = (int)pl->unit_nseg.size(), NC = (int)pl->chunk_u0.size();
    const size_t o_uboff = off; off = align16(off + (U + 1) * 4);
    const size_t o_clo = off; off = align16(off + (NC + 1) * 4);
    const size_t o_uc0 = off; off = align16(off + U * 4);
    const size_t o_cu0 = off; off = align16(off + NC * 4);
    const size_t o_cu1 = off; off = align16(off + NC * 4);
    const size_t o_unseg = off; off = align16(off + U * 4);
    const size_t o_useg = off; off = align16(off + U * 4);
    const size_t o_ent = off; off = align16(off + pl->k2_ent.size() * 4);
    const size_t o_umeta = off; off = align16(off + pl->unit_meta.size() * 4);
    const size_t o_cinfo = off; off = align16(off + pl->chunk_info.size() * 4);
    const size_t o_acinfo = off; off = align16(off + (size_t)pl->alt_nchunks * 16);
    const size_t o_aumeta = off; off = align16(off + (pl->alt_nchunks ? pl->alt_unit_meta.size() * 4 : 0));
    const size_t o_taux = off; off = align16(off + pl->tile_aux.size() * 4);
    const size_t total = off;
    uint8_t *h;
    if (p->host_only) {
        pl->host_buf.resize(total);
        h = pl->host_buf.data();
    } else {
        h = static_cast<uint8_t *>(pl->pin_plan.acquire(total));
        if (!h) return fail(HALO_ENOMEM, "pinned plan staging (%zu bytes)", total);
    }
    auto put = [&](size_t o, const void *src, size_t n) { if (n) memcpy(h + o, src, n); };
    put(o_tiles, pl->tiles.data(), pl->tiles.size() * sizeof(PrefixTile));
    put(o_order, pl->req_order.data(), nreq * 4);
    put(o_nblk, pl->node_blocks.data(), pl->node_blocks.size() * 4);
    put(o_unit, pl->unit_req.data(), nreq * 4);
    put(o_boff, pl->req_blk_off.data(), (nreq + 1) * 4);
    put(o_blk, pl->req_blk.data(), pl->req_blk.size() * 4);
    put(o_nsl, pl->req_nslots.data(), nreq * 4);
    put(o_uboff, pl->unit_boff.data(), (U + 1) * 4);
    put(o_clo, pl->chunk_lo.data(), (NC + 1) * 4);
    put(o_uc0, pl->unit_chunk0.data(), U * 4);
    put(o_cu0, pl->chunk_u0.data(), NC * 4);
    put(o_cu1, pl->chunk_u1.data(), NC * 4);
    put(o_unseg, pl->unit_nseg.data(), U * 4);
    put(o_useg, pl->unit_seg.data(), U * 4);
    put(o_ent, pl->k2_ent.data(), pl->k2_ent.size() * 4);
    put(o_umeta, pl->unit_meta.data(), pl->unit_meta.size() * 4);
    put(o_cinfo, pl->chunk_info.data(), pl->chunk_info.size() * 4);
    if (pl->alt_nchunks) {
        put(o_acinfo, pl->alt_chunk_info.data(), (size_t)pl->alt_nchunks * 16);
        put(o_aumeta, pl->alt_unit_meta.data(), pl->alt_unit_meta.size() * 4);
    }
    put(o_taux, pl->tile_aux.data(), pl->tile_aux.size() * 4);
    if (p->host_only) return HALO_OK;

    if (pl->dbuf_cap < total) {
        if (pl->dbuf) {
            HALO_CUDA(cudaStreamSynchronize(s));
            cudaFree(pl->dbuf);
            pl->dbuf = nullptr;
        }
        const size_t cap = total + total / 2 + 4096;
        HALO_CUDA(cudaMalloc(&pl->dbuf, cap));
        pl->dbuf_cap = cap;
    }
    const size_t part_elems = (size_t)pl->info.max_slots * nreq * p->cfg.num_q_heads * (p->cfg.head_dim + 1);
    if (pl->part_cap < part_elems) {
        if (pl->part) {
            HALO_CUDA(cudaStreamSynchronize(s));
            cudaFree(pl->part);
            pl->part = nullptr;
        }
        const size_t cap = part_elems + part_elems / 4 + 1024;
        HALO_CUDA(cudaMalloc(&pl->part, cap * 4));
        pl->part_cap = cap;
    }
    // K2 scratch, four layer slots (a K2 launch may overlap the previous layer's): stream-K
    // pieces (o in K2's fragment layout, kK2HeadPad heads x d, + (m, l) per head) and parked
    // whole-unit states (g heads x (d + 2)) -- one buffer
    const int gq = p->cfg.num_q_heads / p->cfg.num_kv_heads;
    const int32_t nseg_max = std::max(std::max(pl->nseg_total, pl->alt_nseg_total), 1);
    const size_t seg_slot = (size_t)nseg_max * kK2HeadPad * (p->cfg.head_dim + 2);
    const size_t park_slot = (size_t)U * gq * (p->cfg.head_dim + 2);
    const size_t seg_elems = 4 * (seg_slot + park_slot);
    if (pl->seg_cap < seg_elems) {
        if (pl->segbuf) {
            HALO_CUDA(cudaStreamSynchronize(s));
            cudaFree(pl->segbuf);
            pl->segbuf = nullptr;
        }
        const size_t cap = seg_elems + seg_elems / 4 + 1024;
        HALO_CUDA(cudaMalloc(&pl->segbuf, cap * 4));
        pl->seg_cap = cap;
    }
    // counters: unit arrivals x 4 slots, then dyn claims [4], K1 done [4], K2 done [4]
    const size_t ncount = 4 * ((size_t)U + 2) + 12;
    if (pl->counter_cap < ncount) {
        if (pl->counters) {
            HALO_CUDA(cudaStreamSynchronize(s));
            cudaFree(pl->counters);
            pl->counters = nullptr;
        }
        const size_t cap = ncount + U + 64;
        HALO_CUDA(cudaMalloc(&pl->counters, cap * 4));
        pl->counter_cap = cap;
    }
    HALO_CUDA(cudaMemsetAsync(pl->counters, 0, ncount * 4, s));
    HALO_CUDA(pl->pin_plan.commit(pl->dbuf, total, s));
    uint8_t *d = static_cast<uint8_t *>(pl->dbuf);
    PlanDev &dv = pl->dev;
    dv.tiles = reinterpret_cast<const PrefixTile *>(d + o_tiles);
    dv.req_order = reinterpret_cast<const int32_t *>(d + o_order);
    dv.node_blocks = reinterpret_cast<const int32_t *>(d + o_nblk);
    dv.unit_req = reinterpret_cast<const int32_t *>(d + o_unit);
    dv.req_blk_off = reinterpret_cast<const int32_t *>(d + o_boff);
    dv.req_blk = reinterpret_cast<const uint32_t *>(d + o_blk);
    dv.req_nslots = reinterpret_cast<const int32_t *>(d + o_nsl);
    dv.part_o = pl->part;
    dv.part_lse = pl->part + (size_t)pl->info.max_slots * nreq * p->cfg.num_q_heads * p->cfg.head_dim;
    dv.unit_boff = reinterpret_cast<const int32_t *>(d + o_uboff);
    dv.chunk_lo = reinterpret_cast<const int32_t *>(d + o_clo);
    dv.unit_chunk0 = reinterpret_cast<const int32_t *>(d + o_uc0);
    dv.chunk_u0 = reinterpret_cast<const int32_t *>(d + o_cu0);
    dv.chunk_u1 = reinterpret_cast<const int32_t *>(d + o_cu1);
    dv.unit_nseg = reinterpret_cast<const int32_t *>(d + o_unseg);
    dv.unit_seg = reinterpret_cast<const int32_t *>(d + o_useg);
    dv.unit_count = pl->counters;
    dv.count_slot_stride = U + 2;
    dv.dyn_counter = pl->counters + 4 * (U + 2);
    dv.k1_done = reinterpret_cast<uint32_t *>(pl->counters + 4 * (U + 2) + 4);
    dv.k2_done = reinterpret_cast<uint32_t *>(pl->counters + 4 * (U + 2) + 8);
    dv.dyn_first = pl->dyn_first;
    dv.k2_ent = reinterpret_cast<const uint2 *>(d + o_ent);
    dv.unit_meta = reinterpret_cast<const int4 *>(d + o_umeta);
    dv.chunk_info = reinterpret_cast<const int4 *>(d + o_cinfo);
    dv.alt_nchunks = pl->alt_nchunks;
    dv.alt_chunk_info = reinterpret_cast<const int4 *>(d + o_acinfo);
    dv.alt_unit_meta = reinterpret_cast<const int4 *>(d + o_aumeta);
    dv.tile_aux = reinterpret_cast<const int4 *>(d + o_taux);
    dv.nchunks = NC;
    dv.nblocks = pl->unit_boff.empty() ? 0 : pl->unit_boff.back();
    dv.seg_o = pl->segbuf;
    dv.seg_ml = pl->segbuf + (size_t)nseg_max * kK2HeadPad * p->cfg.head_dim;
    dv.seg_slot_stride = (int64_t)seg_slot;
    dv.park = pl->segbuf + 4 * seg_slot;
    dv.nwarps = k2_sms(pl) * pl->k2_warps;
    dv.k2_warps = pl->k2_warps;
    dv.ntiles = (int32_t)pl->tiles.size();
    dv.nreq = nreq;
    dv.nunits = nreq * p->cfg.num_kv_heads;
    dv.max_slots = pl->info.max_slots;
    return HALO_OK;
}

halo_status run_layer(halo_plan pl, int32_t layer, const void *q, float *out, float *lse,
                      float scale, cudaStream_t s, int mask = 3) {
    halo_pool p = pl->pool;
    if (pl->layout_gen != p->layout_gen)
        return fail(HALO_EBUSY, "stale plan: blocks were given back or a node moved since it was built (re-plan)");
    cudaError_t e;
    if (mask & 1) {
        const CUtensorMap *tq = nullptr;
        if (pl->dev.ntiles > 0 && pl->nreq > 0 && (reinterpret_cast<uintptr_t>(q) & 15) == 0) {
            if (pl->tmap_q_ptr != q || pl->tmap_q_nreq != pl->nreq) {
                pl->tmap_q_ok = make_qmap(p, q, pl->nreq, &pl->tmap_q) == HALO_OK;
                pl->tmap_q_ptr = q;
                pl->tmap_q_nreq = pl->nreq;
            }
            if (pl->tmap_q_ok) tq = &pl->tmap_q;
        }
        e = launch_prefix_attn(&p->tmap_k, &p->tmap_v, &p->tmap_k8, &p->tmap_v8, tq, pl->dev, p->geom, layer, q,
                               scale, s);
        if (e != cudaSuccess) return fail(HALO_ECUDA, "prefix kernel launch: %s", cudaGetErrorString(e));
    }
    if (mask & 2) {
        PlanDev dv = pl->dev;
        if (!(mask & 1) && dv.alt_nchunks > 0) {  // K2 alone: the equal-share schedule
            dv.k2_warps = pl->alt_k2_warps;
            dv.nwarps = k2_sms(pl) * pl->alt_k2_warps;
            dv.chunk_info = dv.alt_chunk_info;
            dv.unit_meta = dv.alt_unit_meta;
            dv.nchunks = dv.alt_nchunks;
            dv.dyn_first = dv.alt_nchunks;
        }
        if (dv.nblocks == 0 && dv.nunits > 0 && dv.max_slots > 0) {
            // no suffix blocks at all (prefill plans whose causal parts ran in K1): K3 alone
            e = launch_merge_only(dv, p->geom, layer, out, lse, s);
            if (e != cudaSuccess) return fail(HALO_ECUDA, "merge kernel launch: %s", cudaGetErrorString(e));
        } else {
            e = launch_suffix_decode(&p->tmap_k, &p->tmap_v, dv, p->geom, layer, q, out, lse, scale, s);
            if (e != cudaSuccess) return fail(HALO_ECUDA, "suffix kernel launch: %s", cudaGetErrorString(e));
        }
    }
    return HALO_OK;
}

// Migration staging buffer (both parities of every transfer's send or receive slice).  A
// grow waits for the previous exchange's last use of the old buffer (mig_done on its stream).
halo_status ensure_mig(halo_pool p, size_t bytes) {
    if (p->mig_cap >= bytes) return HALO_OK;
    if (p->mig_buf) {
        if (p->mig_done) HALO_CUDA(cudaEventSynchronize(p->mig_done));
        HALO_CUDA(cudaFree(p->mig_buf));
        p->mig_buf = nullptr;
        p->mig_cap = 0;
    }
    if (cudaMalloc(&p->mig_buf, bytes) != cudaSuccess) {
        cudaGetLastError();
        p->mig_buf = nullptr;
        return fail(HALO_ENOMEM, "migration staging buffer of %zu bytes", bytes);
    }
    p->mig_cap = bytes;
    return HALO_OK;
}

std::vector<int32_t> token_slots(const std::vector<int32_t> &blocks, int64_t n) {
    std::vector<int32_t> slots(n);
    for (int64_t i = 0; i < n; ++i) slots[i] = blocks[i / kBlockTok] * kBlockTok + (int32_t)(i % kBlockTok);
    return slots;
}

// ---------------------------------------------------------------- host paging
// Host blocks become reusable once the copies enqueued so far have passed (same scheme as
// device blocks: events recorded on every stream that used the pool).
void reclaim_host(halo_pool p, bool wait) {
    for (size_t i = 0; i < p->host_pending.size();) {
        PendingFree &pf = p->host_pending[i];
        bool done = true;
        for (cudaEvent_t e : pf.events) {
            cudaError_t r = wait ? cudaEventSynchronize(e) : cudaEventQuery(e);
            if (r == cudaErrorNotReady) {
                done = false;
                break;
            }
            if (r != cudaSuccess) cudaGetLastError();
        }
        if (!done) {
            ++i;
            continue;
        }
        for (auto it = pf.blocks.rbegin(); it != pf.blocks.rend(); ++it) p->host_free.push_back(*it);
        for (cudaEvent_t e : pf.events) p->event_cache.push_back(e);
        p->host_pending.erase(p->host_pending.begin() + i);
    }
}

halo_status alloc_host_blocks(halo_pool p, int64_t n, std::vector<int32_t> &out) {
    if ((int64_t)p->host_free.size() < n) reclaim_host(p, false);
    if ((int64_t)p->host_free.size() < n) reclaim_host(p, true);
    if ((int64_t)p->host_free.size() < n)
        return fail(HALO_ENOMEM, "host arena out of blocks: need %lld, free %lld", (long long)n,
                    (long long)p->host_free.size());
    for (int64_t i = 0; i < n; ++i) {
        out.push_back(p->host_free.back());
        p->host_free.pop_back();
    }
    return HALO_OK;
}

void release_host_blocks(halo_pool p, std::vector<int32_t> &&blocks) {
    if (blocks.empty()) return;
    if (p->host_only) {
        for (auto it = blocks.rbegin(); it != blocks.rend(); ++it) p->host_free.push_back(*it);
        return;
    }
    PendingFree pf;
    pf.blocks = std::move(blocks);
    for (auto &f : p->streams) {
        cudaEvent_t e = get_event(p);
        if (e && cudaEventRecord(e, f.stream) == cudaSuccess) pf.events.push_back(e);
        else cudaGetLastError();
    }
    p->host_pending.push_back(std::move(pf));
}

// Copy every layer of block list `dev` <-> `host` (same length), K and V, one cudaMemcpyAsync
// per run of blocks consecutive on both sides (a registered node is one run per layer).
halo_status copy_node_blocks(halo_pool p, const std::vector<int32_t> &dev, const std::vector<int32_t> &host,
                             bool to_host, cudaStream_t s) {
    const size_t bb = (size_t)p->cfg.num_kv_heads * kBlockTok * p->cfg.head_dim * 2;  // bytes per block per layer
    const size_t dl = (size_t)p->cfg.capacity_blocks * bb, hl = (size_t)p->host_cap * bb;
    for (int l = 0; l < p->cfg.num_layers; ++l) {
        for (size_t i = 0; i < dev.size();) {
            size_t j = i + 1;
            while (j < dev.size() && dev[j] == dev[j - 1] + 1 && host[j] == host[j - 1] + 1) ++j;
            const size_t n = (j - i) * bb;
            for (int kv = 0; kv < 2; ++kv) {
                uint8_t *d = static_cast<uint8_t *>(kv ? p->v : p->k) + l * dl + (size_t)dev[i] * bb;
                uint8_t *h = static_cast<uint8_t *>(kv ? p->hv : p->hk) + l * hl + (size_t)host[i] * bb;
                HALO_CUDA(cudaMemcpyAsync(to_host ? (void *)h : (void *)d, to_host ? (const void *)d : (const void *)h,
                                          n, to_host ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, s));
            }
            i = j;
        }
    }
    return HALO_OK;
}

halo_status offload_node(halo_pool p, Node &n, cudaStream_t s) {
    std::vector<int32_t> hb;
    halo_status st = alloc_host_blocks(p, (int64_t)n.blocks.size(), hb);
    if (st != HALO_OK) return st;
    if (!p->host_only) {
        st = copy_node_blocks(p, n.blocks, hb, true, s);
        if (st != HALO_OK) {
            for (auto it = hb.rbegin(); it != hb.rend(); ++it) p->host_free.push_back(*it);
            return st;
        }
        note_stream(p, s);
    }
    release_blocks(p, std::move(n.blocks));  // device blocks return once the copy has passed
    n.blocks.clear();
    n.host_blocks = std::move(hb);
    n.on_host = true;
    p->layout_gen++;
    return HALO_OK;
}

}  // namespace

// =====================================================================================
extern "C" {

const char *halo_last_error(void) { return g_err.c_str(); }
int32_t halo_abi_version(void) { return HALO_ABI_VERSION; }

size_t halo_pool_storage_bytes(const halo_pool_config *cfg) { return cfg ? storage_bytes(*cfg) : 0; }

halo_status halo_pool_create(const halo_pool_config *cfg, halo_pool *out) {
    HALO_GUARD_BEGIN
    if (!cfg || !out) return fail(HALO_EINVAL, "null argument");
    const auto &c = *cfg;
    if (c.num_layers < 1 || c.num_kv_heads < 1 || c.num_kv_heads > 64 || c.num_q_heads < 1 ||
        c.num_q_heads % c.num_kv_heads != 0)
        return fail(HALO_EINVAL, "bad head/layer counts");
    const int g = c.num_q_heads / c.num_kv_heads;
    if (g != 1 && g != 2 && g != 4 && g != 8) return fail(HALO_EINVAL, "q heads per kv head must be 1, 2, 4 or 8");
    if (c.head_dim != 64 && c.head_dim != 128) return fail(HALO_EINVAL, "head_dim must be 64 or 128");
    if (c.block_tokens != kBlockTok) return fail(HALO_EINVAL, "block_tokens must be 16");
    if (c.capacity_blocks < 1 || c.capacity_blocks * c.num_kv_heads > (int64_t)kBlkMask + 1 ||
        (int64_t)c.num_layers * c.capacity_blocks >= ((int64_t)1 << 31))
        return fail(HALO_EINVAL, "capacity_blocks out of range");
    if ((c.k_storage == nullptr) != (c.v_storage == nullptr))
        return fail(HALO_EINVAL, "k_storage and v_storage must both be set or both NULL");
    auto *p = new halo_pool_s();
    p->cfg = c;
    p->host_only = c.device < 0;
    p->geom = PoolGeom{c.num_layers, c.num_kv_heads, c.num_q_heads, c.head_dim, c.capacity_blocks, nullptr};
    p->blk_epoch.assign(c.capacity_blocks, 0);
    p->free_list.reserve(c.capacity_blocks);
    for (int64_t b = c.capacity_blocks - 1; b >= 0; --b) p->free_list.push_back((int32_t)b);
    if (!p->host_only) {
        DeviceGuard dg(p);
        int dev_count = 0;
        if (cudaGetDeviceCount(&dev_count) != cudaSuccess || c.device >= dev_count) {
            cudaGetLastError();
            delete p;
            return fail(HALO_EINVAL, "no CUDA device %d", c.device);
        }
        cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, c.device);
        {
            // The library's small per-call device scratch (slot lists, block pairs) comes from
            // cudaMallocAsync; keep up to 1 GiB of freed memory cached in the device's default
            // pool instead of unmapping it at every synchronisation (release threshold 0).
            cudaMemPool_t mp;
            if (cudaDeviceGetDefaultMemPool(&mp, c.device) == cudaSuccess) {
                uint64_t thr = 0;
                cudaMemPoolGetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
                if (thr < (1ull << 30)) {
                    thr = 1ull << 30;
                    cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
                }
            }
            cudaGetLastError();
        }
        const size_t bytes = storage_bytes(c);
        if (c.k_storage) {
            p->k = c.k_storage;
            p->v = c.v_storage;
        } else {
            if (cudaMalloc(&p->k, bytes) != cudaSuccess || cudaMalloc(&p->v, bytes) != cudaSuccess) {
                cudaGetLastError();
                if (p->k) cudaFree(p->k);
                delete p;
                return fail(HALO_ENOMEM, "cudaMalloc of %zu bytes x 2 failed", bytes);
            }
            p->own_storage = true;
        }
        halo_status st = HALO_OK;
        const size_t vbytes = (size_t)c.num_layers * c.capacity_blocks * sizeof(uint64_t);
        if (cudaMalloc(&p->geom.vmax, vbytes) != cudaSuccess) {
            cudaGetLastError();
            p->geom.vmax = nullptr;
            st = fail(HALO_ENOMEM, "cudaMalloc of the V table (%zu bytes) failed", vbytes);
        }
        if (st == HALO_OK && (cudaMemset(p->k, 0, bytes) != cudaSuccess || cudaMemset(p->v, 0, bytes) != cudaSuccess ||
                              cudaMemset(p->geom.vmax, 0, vbytes) != cudaSuccess))
            st = fail(HALO_ECUDA, "cudaMemset of the pool failed");
        if (st == HALO_OK) st = make_tmap(p, p->k, &p->tmap_k, 1);
        if (st == HALO_OK) st = make_tmap(p, p->v, &p->tmap_v, 1);
        if (st == HALO_OK) st = make_tmap(p, p->k, &p->tmap_k8, 8);
        if (st == HALO_OK) st = make_tmap(p, p->v, &p->tmap_v8, 8);
        if (st != HALO_OK) {
            if (p->own_storage) {
                cudaFree(p->k);
                cudaFree(p->v);
            }
            if (p->geom.vmax) cudaFree(p->geom.vmax);
            delete p;
            return st;
        }
    }
    *out = p;
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_pool_destroy(halo_pool p) {
    HALO_GUARD_BEGIN
    if (!p) return fail(HALO_EINVAL, "null pool");
    if (p->plans_alive > 0) return fail(HALO_EBUSY, "%d plan(s) still alive", p->plans_alive);
    if (!p->host_only) {
        DeviceGuard dg(p);
        cudaDeviceSynchronize();
        for (auto &pf : p->pending)
            for (cudaEvent_t e : pf.events) cudaEventDestroy(e);
        for (cudaEvent_t e : p->event_cache) cudaEventDestroy(e);
        for (auto &n : p->nodes)
            if (n.second.ready) cudaEventDestroy(n.second.ready);
        p->pin_up.release();
        for (cudaEvent_t e : p->mig_ev)
            if (e) cudaEventDestroy(e);
        if (p->mig_done) cudaEventDestroy(p->mig_done);
        if (p->comm && nccl().ok) nccl().CommDestroy(p->comm);
        if (p->side) cudaStreamDestroy(p->side);
        if (p->mig_buf) cudaFree(p->mig_buf);
        for (auto &pf : p->host_pending)
            for (cudaEvent_t e : pf.events) cudaEventDestroy(e);
        if (p->hk) cudaFreeHost(p->hk);
        if (p->hv) cudaFreeHost(p->hv);
        if (p->own_storage) {
            cudaFree(p->k);
            cudaFree(p->v);
        }
        if (p->geom.vmax) cudaFree(p->geom.vmax);
    }
    delete p;
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_pool_stats(halo_pool p, int64_t *free_blocks, int64_t *used_blocks) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    { DeviceGuard dg(p); reclaim(p, false); }
    int64_t pend = 0;
    for (auto &pf : p->pending) pend += (int64_t)pf.blocks.size();
    if (free_blocks) *free_blocks = (int64_t)p->free_list.size();
    if (used_blocks) *used_blocks = p->cfg.capacity_blocks - (int64_t)p->free_list.size() - pend;
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_pool_storage(halo_pool p, void **k, void **v) {
    if (check_pool(p)) return HALO_EINVAL;
    if (k) *k = p->k;
    if (v) *v = p->v;
    return HALO_OK;
}

halo_status halo_prefix_register(halo_pool p, int64_t parent, int32_t ntok, const void *k,
                                 const void *v, void *stream, int64_t *node_out) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    if (!node_out || ntok < 1) return fail(HALO_EINVAL, "ntok must be >= 1 and node_out non-null");
    if (parent >= 0 && !p->nodes.count(parent)) return fail(HALO_ENOENT, "unknown parent %lld", (long long)parent);
    if (parent < -1) return fail(HALO_EINVAL, "bad parent id");
    if (!p->host_only && (!k || !v)) return fail(HALO_EINVAL, "null k/v");
    DeviceGuard dg(p);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nblk = ceil_div(ntok, kBlockTok);
    std::vector<int32_t> blocks;
    halo_status st = alloc_blocks(p, nblk, blocks);
    if (st != HALO_OK) return st;
    if (!p->host_only) {
        const size_t bytes = (size_t)p->cfg.num_layers * ntok * p->cfg.num_kv_heads * p->cfg.head_dim * 2;
        std::vector<int32_t> slots = token_slots(blocks, nblk * kBlockTok);
        std::vector<uint32_t> tags = slot_tags(p, slots);
        slots.insert(slots.end(), tags.begin(), tags.end());  // one upload: slots | tags
        Scratch ss, sk, sv;
        const void *dk = nullptr, *dvp = nullptr;
        st = upload(p, slots.data(), slots.size() * 4, s, ss);
        if (st == HALO_OK) st = as_device(k, bytes, s, sk, &dk);
        if (st == HALO_OK) st = as_device(v, bytes, s, sv, &dvp);
        if (st == HALO_OK) {
            const int32_t *ds = (const int32_t *)ss.ptr;
            cudaError_t e = launch_kv_scatter(p->geom, p->k, p->v, dk, dvp, ntok, ds,
                                              (const uint32_t *)(ds + nblk * kBlockTok), ntok,
                                              nblk * kBlockTok - ntok, 0, p->cfg.num_layers, p->num_sms, s);
            if (e != cudaSuccess) st = fail(HALO_ECUDA, "scatter launch: %s", cudaGetErrorString(e));
        }
        if (st != HALO_OK) {
            unalloc_blocks(p, blocks, 0);
            return st;
        }
        note_stream(p, s);
    }
    const int64_t id = p->next_id++;
    Node n;
    n.parent = parent;
    n.ntok = ntok;
    n.blocks = std::move(blocks);
    p->nodes.emplace(id, std::move(n));
    if (parent >= 0) p->nodes[parent].children++;
    *node_out = id;
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_prefix_release(halo_pool p, int64_t node) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    auto it = p->nodes.find(node);
    if (it == p->nodes.end()) return fail(HALO_ENOENT, "unknown node %lld", (long long)node);
    if (it->second.children || it->second.requests)
        return fail(HALO_EBUSY, "node %lld has %d children and %d requests", (long long)node,
                    it->second.children, it->second.requests);
    DeviceGuard dg(p);
    const int64_t parent = it->second.parent;
    release_blocks(p, std::move(it->second.blocks));
    release_host_blocks(p, std::move(it->second.host_blocks));
    if (it->second.ready) p->event_cache.push_back(it->second.ready);
    p->nodes.erase(it);
    if (parent >= 0) p->nodes[parent].children--;
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_prefix_read(halo_pool p, int64_t node, void *k_out, void *v_out, void *stream) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    if (p->host_only) return fail(HALO_EUNSUPPORTED, "host-only pool");
    auto it = p->nodes.find(node);
    if (it == p->nodes.end()) return fail(HALO_ENOENT, "unknown node %lld", (long long)node);
    if (it->second.on_host) return fail(HALO_EBUSY, "node %lld is offloaded: fetch it first", (long long)node);
    if (!k_out || !v_out) return fail(HALO_EINVAL, "null output");
    DeviceGuard dg(p);
    cudaStream_t s = (cudaStream_t)stream;
    halo_status st = wait_ready(p, it->second, s);
    if (st != HALO_OK) return st;
    std::vector<int32_t> slots = token_slots(it->second.blocks, it->second.ntok);
    Scratch ss;
    st = upload(p, slots.data(), slots.size() * 4, s, ss);
    if (st != HALO_OK) return st;
    cudaError_t e = launch_kv_gather(p->geom, p->k, p->v, k_out, v_out, (const int32_t *)ss.ptr,
                                     it->second.ntok, 0, p->cfg.num_layers, p->num_sms, s);
    if (e != cudaSuccess) return fail(HALO_ECUDA, "gather launch: %s", cudaGetErrorString(e));
    note_stream(p, s);
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_node_info(halo_pool p, int64_t node, int64_t *parent, int32_t *ntok, int32_t *nblocks,
                           int32_t *blocks_out) {
    if (check_pool(p)) return HALO_EINVAL;
    auto it = p->nodes.find(node);
    if (it == p->nodes.end()) return fail(HALO_ENOENT, "unknown node %lld", (long long)node);
    if (parent) *parent = it->second.parent;
    if (ntok) *ntok = it->second.ntok;
    if (nblocks) *nblocks = (int32_t)it->second.blocks.size();
    if (blocks_out) memcpy(blocks_out, it->second.blocks.data(), it->second.blocks.size() * 4);
    return HALO_OK;
}

halo_status halo_request_open(halo_pool p, int64_t leaf, int64_t *req_out) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    if (!req_out) return fail(HALO_EINVAL, "null req_out");
    if (leaf < -1) return fail(HALO_EINVAL, "bad leaf id");
    if (leaf >= 0 && !p->nodes.count(leaf)) return fail(HALO_ENOENT, "unknown node %lld", (long long)leaf);
    const int64_t id = p->next_id++;
    Request r;
    r.leaf = leaf;
    p->requests.emplace(id, std::move(r));
    if (leaf >= 0) p->nodes[leaf].requests++;
    *req_out = id;
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_request_close(halo_pool p, int64_t req) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    auto it = p->requests.find(req);
    if (it == p->requests.end()) return fail(HALO_ENOENT, "unknown request %lld", (long long)req);
    DeviceGuard dg(p);
    const int64_t leaf = it->second.leaf;
    release_blocks(p, std::move(it->second.blocks));
    p->requests.erase(it);
    if (leaf >= 0) p->nodes[leaf].requests--;
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_request_info(halo_pool p, int64_t req, int64_t *leaf, int32_t *suffix_len, int32_t *nblocks) {
    if (check_pool(p)) return HALO_EINVAL;
    auto it = p->requests.find(req);
    if (it == p->requests.end()) return fail(HALO_ENOENT, "unknown request %lld", (long long)req);
    if (leaf) *leaf = it->second.leaf;
    if (suffix_len) *suffix_len = it->second.len;
    if (nblocks) *nblocks = (int32_t)it->second.blocks.size();
    return HALO_OK;
}

// Host half of an append: validate (repeated ids allowed), allocate the new blocks and the
// pool slot of every new token in input order.  Nothing is committed: `work` holds the new
// (len, blocks) of every touched request; append_commit applies it, and on a later failure
// unalloc_blocks(fresh) undoes the allocation.
struct AppendWork {
    std::vector<int32_t> slots, fresh;
    std::unordered_map<int64_t, std::pair<int32_t, std::vector<int32_t>>> req;
    int64_t total = 0;
};

halo_status append_prepare(halo_pool p, int32_t nreq, const int64_t *reqs, const int32_t *ntok, AppendWork &w) {
    if (nreq < 0 || (nreq > 0 && (!reqs || !ntok))) return fail(HALO_EINVAL, "bad request list");
    std::unordered_map<int64_t, std::pair<int32_t, int64_t>> sim;  // id -> (len, nblocks)
    int64_t new_blocks = 0;
    w.total = 0;
    for (int i = 0; i < nreq; ++i) {
        auto it = p->requests.find(reqs[i]);
        if (it == p->requests.end()) return fail(HALO_ENOENT, "unknown request %lld", (long long)reqs[i]);
        if (ntok[i] < 0) return fail(HALO_EINVAL, "negative token count");
        auto f = sim.find(reqs[i]);
        if (f == sim.end())
            f = sim.emplace(reqs[i], std::make_pair(it->second.len, (int64_t)it->second.blocks.size())).first;
        const int64_t len = (int64_t)f->second.first + ntok[i];
        if (len > INT32_MAX / 2) return fail(HALO_EINVAL, "suffix too long");
        const int64_t need = ceil_div(len, kBlockTok);
        if (need > f->second.second) {
            new_blocks += need - f->second.second;
            f->second.second = need;
        }
        f->second.first = (int32_t)len;
        w.total += ntok[i];
    }
    if (w.total == 0) return HALO_OK;
    halo_status st = alloc_blocks(p, new_blocks, w.fresh);
    if (st != HALO_OK) return st;
    w.slots.reserve(w.total);
    size_t fi = 0;
    for (int i = 0; i < nreq; ++i) {
        auto r = w.req.find(reqs[i]);
        if (r == w.req.end()) {
            const Request &rq = p->requests[reqs[i]];
            r = w.req.emplace(reqs[i], std::make_pair(rq.len, rq.blocks)).first;
        }
        for (int32_t t = 0; t < ntok[i]; ++t) {
            const int32_t pos = r->second.first++;
            if (pos % kBlockTok == 0 && pos / kBlockTok >= (int32_t)r->second.second.size())
                r->second.second.push_back(w.fresh[fi++]);
            w.slots.push_back(r->second.second[pos / kBlockTok] * kBlockTok + pos % kBlockTok);
        }
    }
    return HALO_OK;
}

void append_commit(halo_pool p, AppendWork &w) {
    for (auto &r : w.req) {
        Request &rq = p->requests[r.first];
        rq.len = r.second.first;
        rq.blocks = std::move(r.second.second);
    }
}

halo_status halo_suffix_append(halo_pool p, int32_t nreq, const int64_t *reqs, const int32_t *ntok,
                               const void *k, const void *v, void *stream) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    if (nreq < 0 || (nreq > 0 && (!reqs || !ntok))) return fail(HALO_EINVAL, "bad request list");
    for (int i = 0; i < nreq; ++i)
        if (ntok[i] > 0 && !p->host_only && (!k || !v)) return fail(HALO_EINVAL, "null k/v");
    DeviceGuard dg(p);
    AppendWork w;
    halo_status st = append_prepare(p, nreq, reqs, ntok, w);
    if (st != HALO_OK || w.total == 0) return st;
    if (!p->host_only) {
        cudaStream_t s = (cudaStream_t)stream;
        const size_t bytes = (size_t)p->cfg.num_layers * w.total * p->cfg.num_kv_heads * p->cfg.head_dim * 2;
        Scratch ss, sk, sv;
        const void *dk = nullptr, *dvp = nullptr;
        std::vector<int32_t> st_buf = w.slots;
        std::vector<uint32_t> tags = slot_tags(p, w.slots);
        st_buf.insert(st_buf.end(), tags.begin(), tags.end());  // slots | tags
        st = upload(p, st_buf.data(), st_buf.size() * 4, s, ss);
        if (st == HALO_OK) st = as_device(k, bytes, s, sk, &dk);
        if (st == HALO_OK) st = as_device(v, bytes, s, sv, &dvp);
        if (st == HALO_OK) {
            const int32_t *ds = (const int32_t *)ss.ptr;
            cudaError_t e = launch_kv_scatter(p->geom, p->k, p->v, dk, dvp, w.total, ds,
                                              (const uint32_t *)(ds + w.total), w.total, 0, 0,
                                              p->cfg.num_layers, p->num_sms, s);
            if (e != cudaSuccess) st = fail(HALO_ECUDA, "scatter launch: %s", cudaGetErrorString(e));
        }
        if (st != HALO_OK) {
            unalloc_blocks(p, w.fresh, 0);
            return st;
        }
        note_stream(p, s);
    }
    append_commit(p, w);
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_suffix_truncate(halo_pool p, int32_t nreq, const int64_t *reqs, const int32_t *ntok) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    if (nreq < 0 || (nreq > 0 && (!reqs || !ntok))) return fail(HALO_EINVAL, "bad request list");
    std::unordered_map<int64_t, int32_t> len;
    for (int i = 0; i < nreq; ++i) {
        auto it = p->requests.find(reqs[i]);
        if (it == p->requests.end()) return fail(HALO_ENOENT, "unknown request %lld", (long long)reqs[i]);
        auto f = len.emplace(reqs[i], it->second.len).first;
        if (ntok[i] < 0 || ntok[i] > f->second) return fail(HALO_EINVAL, "truncate count out of range");
        f->second -= ntok[i];
    }
    DeviceGuard dg(p);
    for (auto &l : len) {
        Request &r = p->requests[l.first];
        r.len = l.second;
        const size_t keep = (size_t)ceil_div(r.len, kBlockTok);
        if (r.blocks.size() > keep) {
            std::vector<int32_t> drop(r.blocks.begin() + keep, r.blocks.end());
            r.blocks.resize(keep);
            release_blocks(p, std::move(drop));
        }
    }
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_decode_plan(halo_pool p, int32_t nreq, const int64_t *reqs, const halo_plan_options *opt,
                             void *stream, halo_plan *inout) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    if (!inout || nreq < 1 || !reqs) return fail(HALO_EINVAL, "need nreq >= 1, reqs and a plan slot");
    if (*inout && (*inout)->pool != p) return fail(HALO_EINVAL, "plan belongs to another pool");
    if (opt && (opt->force_splits < 0)) return fail(HALO_EINVAL, "bad plan options");
    DeviceGuard dg(p);
    const bool fresh = *inout == nullptr;
    halo_plan pl = fresh ? new halo_plan_s() : *inout;
    pl->pool = p;
    pl->opt = opt ? *opt : halo_plan_options{};
    halo_status st = build_plan(pl, nreq, reqs);
    if (st == HALO_OK) st = upload_plan(pl, (cudaStream_t)stream);
    if (st != HALO_OK) {
        if (fresh) {
            if (pl->dbuf) cudaFree(pl->dbuf);
            if (pl->part) cudaFree(pl->part);
            if (pl->segbuf) cudaFree(pl->segbuf);
            if (pl->counters) cudaFree(pl->counters);
            pl->pin_plan.release();
            delete pl;
        }
        return st;
    }
    if (fresh) {
        p->plans_alive++;
        *inout = pl;
    }
    note_stream(p, (cudaStream_t)stream);
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_prefill_plan(halo_pool p, int32_t nreq, const int64_t *reqs, const int32_t *ntok,
                              const halo_plan_options *opt, void *stream, halo_plan *inout) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    if (!inout || nreq < 1 || !reqs || !ntok) return fail(HALO_EINVAL, "need nreq >= 1, reqs, ntok and a plan slot");
    if (*inout && (*inout)->pool != p) return fail(HALO_EINVAL, "plan belongs to another pool");
    if (opt && (opt->force_splits < 0)) return fail(HALO_EINVAL, "bad plan options");
    // one virtual request per new token: token t of request i sees the request's prefix path
    // and the first (len - ntok[i] + t + 1) suffix tokens (causal within the prompt)
    std::vector<Request> virt;
    int64_t total = 0;
    for (int i = 0; i < nreq; ++i) {
        auto it = p->requests.find(reqs[i]);
        if (it == p->requests.end()) return fail(HALO_ENOENT, "unknown request id %lld", (long long)reqs[i]);
        const Request &r = it->second;
        if (ntok[i] < 1 || ntok[i] > r.len)
            return fail(HALO_EINVAL, "request %lld: %d new tokens but a %d-token suffix", (long long)reqs[i],
                        ntok[i], r.len);
        total += ntok[i];
        if (total > INT32_MAX / 64) return fail(HALO_EINVAL, "too many prefill tokens");
    }
    virt.reserve(total);
    std::vector<CausalGroup> groups;
    for (int i = 0; i < nreq; ++i) {
        const Request &r = p->requests[reqs[i]];
        groups.push_back({(int32_t)virt.size(), ntok[i], r.len, &r.blocks});
        for (int32_t t = 0; t < ntok[i]; ++t) {
            Request v;
            v.leaf = r.leaf;
            v.len = r.len - ntok[i] + t + 1;
            v.blocks.assign(r.blocks.begin(), r.blocks.begin() + ceil_div(v.len, kBlockTok));
            virt.push_back(std::move(v));
        }
    }
    DeviceGuard dg(p);
    const bool fresh = *inout == nullptr;
    halo_plan pl = fresh ? new halo_plan_s() : *inout;
    pl->pool = p;
    pl->opt = opt ? *opt : halo_plan_options{};
    halo_status st = build_plan(pl, (int32_t)total, nullptr, &virt, &groups);
    if (st == HALO_OK) st = upload_plan(pl, (cudaStream_t)stream);
    if (st != HALO_OK) {
        if (fresh) {
            if (pl->dbuf) cudaFree(pl->dbuf);
            if (pl->part) cudaFree(pl->part);
            if (pl->segbuf) cudaFree(pl->segbuf);
            if (pl->counters) cudaFree(pl->counters);
            pl->pin_plan.release();
            delete pl;
        }
        return st;
    }
    if (fresh) {
        p->plans_alive++;
        *inout = pl;
    }
    note_stream(p, (cudaStream_t)stream);
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_decode_run(halo_plan pl, int32_t layer, const void *q, float *out, float *lse, float scale,
                            void *stream) {
    HALO_GUARD_BEGIN
    if (!pl) return fail(HALO_EINVAL, "null plan");
    halo_pool p = pl->pool;
    if (p->host_only) return fail(HALO_EUNSUPPORTED, "compute on a host-only pool");
    if (layer < 0 || layer >= p->cfg.num_layers) return fail(HALO_EINVAL, "layer out of range");
    if (!q || !out) return fail(HALO_EINVAL, "null q/out");
    if (!(scale > 0.f)) scale = 1.0f / sqrtf((float)p->cfg.head_dim);
    DeviceGuard dg(p);
    // the stream now reads pool blocks: later frees wait for it (host bookkeeping only, so
    // this is safe under stream capture)
    note_stream(p, (cudaStream_t)stream);
    return run_layer(pl, layer, q, out, lse, scale, (cudaStream_t)stream);
    HALO_GUARD_END
}

halo_status halo_decode_run_stages(halo_plan pl, int32_t layer, int32_t mask, const void *q, float *out,
                                   float *lse, float scale, void *stream) {
    HALO_GUARD_BEGIN
    if (!pl) return fail(HALO_EINVAL, "null plan");
    halo_pool p = pl->pool;
    if (p->host_only) return fail(HALO_EUNSUPPORTED, "compute on a host-only pool");
    if (layer < 0 || layer >= p->cfg.num_layers) return fail(HALO_EINVAL, "layer out of range");
    if (mask < 0 || mask > 3) return fail(HALO_EINVAL, "bad stage mask");
    if (!q || ((mask & 2) && !out)) return fail(HALO_EINVAL, "null q/out");
    if (!(scale > 0.f)) scale = 1.0f / sqrtf((float)p->cfg.head_dim);
    DeviceGuard dg(p);
    note_stream(p, (cudaStream_t)stream);
    return run_layer(pl, layer, q, out, lse, scale, (cudaStream_t)stream, mask);
    HALO_GUARD_END
}

halo_status halo_decode_layers(halo_plan pl, int32_t nlayers, const void *q, float *out, float *lse, float scale,
                               void *stream) {
    HALO_GUARD_BEGIN
    if (!pl) return fail(HALO_EINVAL, "null plan");
    halo_pool p = pl->pool;
    if (p->host_only) return fail(HALO_EUNSUPPORTED, "compute on a host-only pool");
    if (nlayers < 1 || nlayers > p->cfg.num_layers) return fail(HALO_EINVAL, "nlayers out of range");
    if (!q || !out) return fail(HALO_EINVAL, "null q/out");
    if (!(scale > 0.f)) scale = 1.0f / sqrtf((float)p->cfg.head_dim);
    DeviceGuard dg(p);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t rows = (size_t)pl->nreq * p->cfg.num_q_heads;
    const size_t q_layer = rows * p->cfg.head_dim;  // elements
    const size_t o_layer = rows * p->cfg.head_dim;
    const void *dq = q;
    float *dout = out, *dlse = lse;
    const bool q_host = !is_device_ptr(q), o_host = !is_device_ptr(out), l_host = lse && !is_device_ptr(lse);
    auto grow = [&](void **buf, size_t *cap, size_t bytes) -> halo_status {
        if (*cap >= bytes) return HALO_OK;
        if (*buf) {
            HALO_CUDA(cudaStreamSynchronize(s));
            cudaFree(*buf);
            *buf = nullptr;
        }
        HALO_CUDA(cudaMalloc(buf, bytes));
        *cap = bytes;
        return HALO_OK;
    };
    halo_status st;
    if (q_host) {
        if ((st = grow(&pl->q_stage, &pl->q_stage_cap, q_layer * nlayers * 2)) != HALO_OK) return st;
        HALO_CUDA(cudaMemcpyAsync(pl->q_stage, q, q_layer * nlayers * 2, cudaMemcpyHostToDevice, s));
        dq = pl->q_stage;
    }
    if (o_host) {
        if ((st = grow((void **)&pl->o_stage, &pl->o_stage_cap, o_layer * nlayers * 4)) != HALO_OK) return st;
        dout = pl->o_stage;
    }
    if (l_host) {
        if ((st = grow((void **)&pl->l_stage, &pl->l_stage_cap, rows * nlayers * 4)) != HALO_OK) return st;
        dlse = pl->l_stage;
    }
    note_stream(p, s);
    for (int l = 0; l < nlayers; ++l) {
        st = run_layer(pl, l, static_cast<const uint16_t *>(dq) + q_layer * l, dout + o_layer * l,
                       dlse ? dlse + rows * l : nullptr, scale, s);
        if (st != HALO_OK) return st;
    }
    if (q_host && pl->ev_used[0]) {
        // the input staging's buffer 0 was read by these layers: halo_decode_step's next upload
        // into it (double-buffered staging) waits for them
        HALO_CUDA(cudaEventRecord(pl->ev_used[0], s));
        pl->ev_used_rec[0] = true;
    }
    if (o_host) HALO_CUDA(cudaMemcpyAsync(out, dout, o_layer * nlayers * 4, cudaMemcpyDeviceToHost, s));
    if (l_host) HALO_CUDA(cudaMemcpyAsync(lse, dlse, rows * nlayers * 4, cudaMemcpyDeviceToHost, s));
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_decode_step(halo_pool p, int32_t nreq, const int64_t *reqs, const void *k_new,
                             const void *v_new, const void *q, float *out, float *lse, float scale,
                             const halo_plan_options *opt, void *stream, halo_plan *inout) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    if (p->host_only) return fail(HALO_EUNSUPPORTED, "compute on a host-only pool");
    if (!inout || nreq < 1 || !reqs) return fail(HALO_EINVAL, "need nreq >= 1, reqs and a plan slot");
    if (!k_new || !v_new || !q || !out) return fail(HALO_EINVAL, "null k/v/q/out");
    if (*inout && (*inout)->pool != p) return fail(HALO_EINVAL, "plan belongs to another pool");
    if (!(scale > 0.f)) scale = 1.0f / sqrtf((float)p->cfg.head_dim);
    DeviceGuard dg(p);
    cudaStream_t s = (cudaStream_t)stream;
    const int L = p->cfg.num_layers, Hq = p->cfg.num_q_heads, Hkv = p->cfg.num_kv_heads, D = p->cfg.head_dim;
    // 1. host bookkeeping of the append (one token per request), then the plan
    std::vector<int32_t> ones(nreq, 1);
    AppendWork w;
    halo_status st = append_prepare(p, nreq, reqs, ones.data(), w);
    if (st != HALO_OK) return st;
    std::vector<std::pair<int64_t, std::pair<int32_t, std::vector<int32_t>>>> undo;
    for (auto &r : w.req) undo.push_back({r.first, {p->requests[r.first].len, p->requests[r.first].blocks}});
    append_commit(p, w);
    auto rollback = [&]() {
        for (auto &u : undo) {
            Request &rq = p->requests[u.first];
            rq.len = u.second.first;
            rq.blocks = u.second.second;
        }
        unalloc_blocks(p, w.fresh, 0);
    };
    st = halo_decode_plan(p, nreq, reqs, opt, stream, inout);
    if (st != HALO_OK) {
        rollback();
        return st;
    }
    halo_plan pl = *inout;
    const size_t kv_layer = (size_t)nreq * Hkv * D;     // elements of one layer's new K (or V)
    const size_t q_layer = (size_t)nreq * Hq * D, rows = (size_t)nreq * Hq;
    const bool kv_host = !is_device_ptr(k_new) || !is_device_ptr(v_new);
    const bool q_host = !is_device_ptr(q), o_host = !is_device_ptr(out), l_host = lse && !is_device_ptr(lse);
    // 2. streams, events and staging (grown once)
    auto grow = [&](void **buf, size_t *cap, size_t bytes) -> halo_status {
        if (*cap >= bytes) return HALO_OK;
        if (*buf) {
            HALO_CUDA(cudaDeviceSynchronize());
            cudaFree(*buf);
            *buf = nullptr;
        }
        HALO_CUDA(cudaMalloc(buf, bytes));
        *cap = bytes;
        return HALO_OK;
    };
    // everything that can fail before the first launch; on failure the append is rolled back
    // (the pool is unchanged) and the rebuilt plan is marked stale
    auto stage = [&]() -> halo_status {
        if (!pl->h2d) {
            HALO_CUDA(cudaStreamCreateWithFlags(&pl->h2d, cudaStreamNonBlocking));
            HALO_CUDA(cudaStreamCreateWithFlags(&pl->d2h, cudaStreamNonBlocking));
            HALO_CUDA(cudaEventCreateWithFlags(&pl->ev_step, cudaEventDisableTiming));
            HALO_CUDA(cudaEventCreateWithFlags(&pl->ev_copied, cudaEventDisableTiming));
            for (int b = 0; b < 2; ++b) HALO_CUDA(cudaEventCreateWithFlags(&pl->ev_used[b], cudaEventDisableTiming));
        }
        while ((int)pl->ev_in.size() < L) {
            cudaEvent_t a, b;
            HALO_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
            HALO_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
            pl->ev_in.push_back(a);
            pl->ev_out.push_back(b);
        }
        if (kv_host && (st = grow(&pl->kv_stage, &pl->kv_stage_cap, 2 * (2 * kv_layer * L * 2))) != HALO_OK) return st;
        if (q_host && (st = grow(&pl->q_stage, &pl->q_stage_cap, 2 * (q_layer * L * 2))) != HALO_OK) return st;
        if (o_host && (st = grow((void **)&pl->o_stage, &pl->o_stage_cap, q_layer * L * 4)) != HALO_OK) return st;
        if (l_host && (st = grow((void **)&pl->l_stage, &pl->l_stage_cap, rows * L * 4)) != HALO_OK) return st;
        if ((st = grow((void **)&pl->slot_stage, &pl->slot_stage_cap, w.slots.size() * 8)) != HALO_OK) return st;
        {
            void *hs = pl->pin_slots.acquire(w.slots.size() * 8);  // slots | V-table tags
            if (!hs) return fail(HALO_ENOMEM, "pinned slot staging");
            memcpy(hs, w.slots.data(), w.slots.size() * 4);
            uint32_t *ht = static_cast<uint32_t *>(hs) + w.slots.size();
            for (size_t i = 0; i < w.slots.size(); ++i) ht[i] = p->blk_epoch[w.slots[i] / kBlockTok];
            HALO_CUDA(pl->pin_slots.commit(pl->slot_stage, w.slots.size() * 8, s));
        }
        return HALO_OK;
    };
    if ((st = stage()) != HALO_OK) {
        rollback();
        p->layout_gen++;
        return st;
    }
    const uint32_t *slot_tags_dev = reinterpret_cast<const uint32_t *>(pl->slot_stage + w.slots.size());
    // 3. pipeline: H2D (k, v, q) on the h2d stream in chunks of kH2DLayers layers, all issued
    //    up front | K5 append + K1 + K2/K3 of layer l on `stream` (waits for its chunk) | D2H
    //    (out, lse) on the d2h stream in chunks of kD2HLayers layers.  Chunk sizes measured on
    //    B200 + PCIe host (tools/e2e_pipe_probe.py, C1): per-layer copies 4.0 ms/step, H2D x4 +
    //    D2H x2 3.07 ms/step (both directions share ~89 GB/s; small D2H chunks start the
    //    output stream early, larger H2D chunks cut the per-copy overhead).  The input staging
    //    is double-buffered: this step's uploads wait only for the compute of the step that
    //    last read the same buffer (two calls ago), so they overlap the previous step's tail
    //    (its last layers and downloads) -- the host link then stays busy in both directions.
    constexpr int kH2DLayers = 4, kD2HLayers = 2;
    const int par = pl->e2e_par;
    pl->e2e_par ^= 1;
    HALO_CUDA(cudaEventRecord(pl->ev_step, s));
    if (pl->ev_used_rec[par]) HALO_CUDA(cudaStreamWaitEvent(pl->h2d, pl->ev_used[par], 0));
    HALO_CUDA(cudaStreamWaitEvent(pl->d2h, pl->ev_step, 0));
    uint16_t *sk = kv_host ? static_cast<uint16_t *>(pl->kv_stage) + par * (2 * kv_layer * L) : nullptr;
    uint16_t *sv = sk ? sk + kv_layer * L : nullptr;
    uint16_t *sq = q_host ? static_cast<uint16_t *>(pl->q_stage) + par * (q_layer * L) : nullptr;
    for (int l = 0; l < L; l += kH2DLayers) {
        const int n = std::min(kH2DLayers, L - l);
        if (kv_host) {
            HALO_CUDA(cudaMemcpyAsync(sk + kv_layer * l, static_cast<const uint16_t *>(k_new) + kv_layer * l,
                                      kv_layer * 2 * n, cudaMemcpyHostToDevice, pl->h2d));
            HALO_CUDA(cudaMemcpyAsync(sv + kv_layer * l, static_cast<const uint16_t *>(v_new) + kv_layer * l,
                                      kv_layer * 2 * n, cudaMemcpyHostToDevice, pl->h2d));
        }
        if (q_host)
            HALO_CUDA(cudaMemcpyAsync(sq + q_layer * l, static_cast<const uint16_t *>(q) + q_layer * l,
                                      q_layer * 2 * n, cudaMemcpyHostToDevice, pl->h2d));
        HALO_CUDA(cudaEventRecord(pl->ev_in[l], pl->h2d));
    }
    const uint16_t *dk = kv_host ? sk : static_cast<const uint16_t *>(k_new);
    const uint16_t *dv = kv_host ? sv : static_cast<const uint16_t *>(v_new);
    const uint16_t *dq = q_host ? sq : static_cast<const uint16_t *>(q);
    float *dout = o_host ? pl->o_stage : out;
    float *dlse = l_host ? pl->l_stage : lse;
    if (!kv_host) {  // device-resident new K/V: one K5 launch appends every layer
        cudaError_t e = launch_kv_scatter(p->geom, p->k, p->v, dk, dv, nreq, pl->slot_stage, slot_tags_dev,
                                          nreq, 0, 0, L, p->num_sms, s);
        if (e != cudaSuccess) return fail(HALO_ECUDA, "append launch: %s", cudaGetErrorString(e));
    }
    for (int l = 0; l < L; ++l) {
        if (l % kH2DLayers == 0) HALO_CUDA(cudaStreamWaitEvent(s, pl->ev_in[l], 0));
        if (kv_host) {  // host K/V: append layer l once its copy has landed
            cudaError_t e = launch_kv_scatter(p->geom, p->k, p->v, dk + kv_layer * l, dv + kv_layer * l, nreq,
                                              pl->slot_stage, slot_tags_dev, nreq, 0, l, l + 1, p->num_sms, s);
            if (e != cudaSuccess) return fail(HALO_ECUDA, "append launch: %s", cudaGetErrorString(e));
        }
        st = run_layer(pl, l, dq + q_layer * l, dout + q_layer * l, dlse ? dlse + rows * l : nullptr, scale, s);
        if (st != HALO_OK) return st;
        if ((o_host || l_host) && (l % kD2HLayers == kD2HLayers - 1 || l == L - 1)) {
            const int l0 = l - l % kD2HLayers, n = l - l0 + 1;
            HALO_CUDA(cudaEventRecord(pl->ev_out[l], s));
            HALO_CUDA(cudaStreamWaitEvent(pl->d2h, pl->ev_out[l], 0));
            if (o_host)
                HALO_CUDA(cudaMemcpyAsync(out + q_layer * l0, dout + q_layer * l0, q_layer * 4 * n,
                                          cudaMemcpyDeviceToHost, pl->d2h));
            if (l_host)
                HALO_CUDA(cudaMemcpyAsync(lse + rows * l0, dlse + rows * l0, rows * 4 * n, cudaMemcpyDeviceToHost,
                                          pl->d2h));
        }
    }
    // the compute of this step has read the input staging buffer `par`
    HALO_CUDA(cudaEventRecord(pl->ev_used[par], s));
    pl->ev_used_rec[par] = true;
    // the step is complete in `stream` order once the last download has landed
    HALO_CUDA(cudaEventRecord(pl->ev_copied, pl->d2h));
    HALO_CUDA(cudaStreamWaitEvent(s, pl->ev_copied, 0));
    note_stream(p, s);
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_plan_get_info(halo_plan pl, halo_plan_info *info) {
    if (!pl || !info) return fail(HALO_EINVAL, "null argument");
    *info = pl->info;
    return HALO_OK;
}

halo_status halo_plan_export(halo_plan pl, int32_t which, void *dst, int64_t cap, int64_t *n) {
    if (!pl || !n) return fail(HALO_EINVAL, "null argument");
    const void *src = nullptr;
    int64_t cnt = 0;
    switch (which) {
        case 0: src = pl->req_order.data(); cnt = (int64_t)pl->req_order.size(); break;
        case 1: src = pl->tiles.data(); cnt = (int64_t)pl->tiles.size() * 8; break;
        case 2: src = pl->req_nslots.data(); cnt = (int64_t)pl->req_nslots.size(); break;
        case 3: src = pl->unit_req.data(); cnt = (int64_t)pl->unit_req.size(); break;
        case 4: src = pl->req_blk_off.data(); cnt = (int64_t)pl->req_blk_off.size(); break;
        case 5: src = pl->req_blk.data(); cnt = (int64_t)pl->req_blk.size(); break;
        case 6: src = pl->unit_boff.data(); cnt = (int64_t)pl->unit_boff.size(); break;
        case 7: src = pl->chunk_u0.data(); cnt = (int64_t)pl->chunk_u0.size(); break;
        case 8: src = pl->chunk_u1.data(); cnt = (int64_t)pl->chunk_u1.size(); break;
        case 9: src = pl->unit_nseg.data(); cnt = (int64_t)pl->unit_nseg.size(); break;
        case 10: src = pl->chunk_lo.data(); cnt = (int64_t)pl->chunk_lo.size(); break;
        default: return fail(HALO_EINVAL, "unknown export %d", which);
    }
    *n = cnt;
    if (dst && cap > 0) memcpy(dst, src, (size_t)std::min(cap, cnt) * 4);
    return HALO_OK;
}

halo_status halo_plan_destroy(halo_plan pl) {
    HALO_GUARD_BEGIN
    if (!pl) return fail(HALO_EINVAL, "null plan");
    halo_pool p = pl->pool;
    {
        DeviceGuard dg(p);
        if (pl->dbuf) cudaFree(pl->dbuf);
        if (pl->part) cudaFree(pl->part);
        if (pl->segbuf) cudaFree(pl->segbuf);
        if (pl->counters) cudaFree(pl->counters);
        if (pl->q_stage) cudaFree(pl->q_stage);
        if (pl->o_stage) cudaFree(pl->o_stage);
        if (pl->l_stage) cudaFree(pl->l_stage);
        pl->pin_plan.release();
        pl->pin_slots.release();
        if (pl->kv_stage) cudaFree(pl->kv_stage);
        if (pl->slot_stage) cudaFree(pl->slot_stage);
        for (cudaEvent_t e : pl->ev_in) cudaEventDestroy(e);
        for (cudaEvent_t e : pl->ev_out) cudaEventDestroy(e);
        if (pl->ev_step) cudaEventDestroy(pl->ev_step);
        if (pl->ev_copied) cudaEventDestroy(pl->ev_copied);
        for (int b = 0; b < 2; ++b)
            if (pl->ev_used[b]) cudaEventDestroy(pl->ev_used[b]);
        if (pl->h2d) cudaStreamDestroy(pl->h2d);
        if (pl->d2h) cudaStreamDestroy(pl->d2h);
    }
    p->plans_alive--;
    delete pl;
    return HALO_OK;
    HALO_GUARD_END
}

// ------------------------------------------------------------------ migration
halo_status halo_comm_unique_id(void *id_out) {
    if (!id_out) return fail(HALO_EINVAL, "null id");
    ncclUniqueId id;
    HALO_NCCL(nccl().GetUniqueId(&id));
    memcpy(id_out, &id, sizeof id);
    return HALO_OK;
}

halo_status halo_comm_init_config(halo_pool p, const void *id, int32_t nranks, int32_t rank,
                                  const halo_comm_config *cfg) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    if (p->host_only) return fail(HALO_EUNSUPPORTED, "host-only pool");
    if (!id || nranks < 1 || rank < 0 || rank >= nranks) return fail(HALO_EINVAL, "bad communicator arguments");
    if (p->comm) return fail(HALO_EBUSY, "communicator already initialised");
    halo_comm_config c{};
    if (cfg) c = *cfg;
    if (c.chunk_bytes <= 0) c.chunk_bytes = (int64_t)32 << 20;
    if (c.copy_ctas <= 0) c.copy_ctas = 8 * p->num_sms;
    DeviceGuard dg(p);
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof uid);
    if (c.max_ctas > 0) {
        if (!nccl().CommInitRankConfig) return fail(HALO_ENCCL, "ncclCommInitRankConfig unavailable");
        ncclConfig_t nc = NCCL_CONFIG_INITIALIZER;
        nc.maxCTAs = c.max_ctas;
        nc.minCTAs = 1;
        HALO_NCCL(nccl().CommInitRankConfig(&p->comm, nranks, uid, rank, &nc));
    } else {
        HALO_NCCL(nccl().CommInitRank(&p->comm, nranks, uid, rank));
    }
    p->nranks = nranks;
    p->rank = rank;
    p->mig_cfg = c;
    if (!p->side) HALO_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
    for (auto &e : p->mig_ev)
        if (!e) HALO_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (!p->mig_done) HALO_CUDA(cudaEventCreateWithFlags(&p->mig_done, cudaEventDisableTiming));
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_comm_init(halo_pool p, const void *id, int32_t nranks, int32_t rank) {
    return halo_comm_init_config(p, id, nranks, rank, nullptr);
}

namespace {

// One transfer of an exchange: a send (pack + ncclSend) or a receive (ncclRecv + unpack).
struct Xfer {
    bool send;
    int32_t peer;
    int64_t nblk, items, nchunks;
    const std::vector<int32_t> *blocks;  // pool blocks in token order (source or destination)
    int64_t dev_off;                     // offset of the block list in the uploaded array
    size_t slice;                        // buffer bytes per parity
    size_t buf_off;                      // offset of the parity-0 slice
};

}  // namespace

halo_status halo_migrate_exchange(halo_pool p, int32_t nsend, const halo_migrate_send_op *sends, int32_t nrecv,
                                  const halo_migrate_recv_op *recvs, void *stream, int64_t *nodes_out) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    if (!p->comm) return fail(HALO_ENCCL, "no communicator (halo_comm_init)");
    if (nsend < 0 || nrecv < 0 || (nsend && !sends) || (nrecv && (!recvs || !nodes_out)))
        return fail(HALO_EINVAL, "bad op arrays");
    if (nsend + nrecv == 0) return HALO_OK;
    // ---- validation (nothing changes on error)
    std::vector<int64_t> moved;
    std::vector<int32_t> self_send_tok, self_recv_tok;
    for (int32_t i = 0; i < nsend; ++i) {
        const auto &o = sends[i];
        auto it = p->nodes.find(o.node);
        if (it == p->nodes.end()) return fail(HALO_ENOENT, "send %d: unknown node %lld", i, (long long)o.node);
        if (it->second.on_host) return fail(HALO_EBUSY, "send %d: node %lld is offloaded: fetch it first", i, (long long)o.node);
        if (o.peer < 0 || o.peer >= p->nranks) return fail(HALO_EINVAL, "send %d: bad peer %d", i, o.peer);
        if (o.mode != 0 && o.mode != 1) return fail(HALO_EINVAL, "send %d: mode must be 0 (MOVE) or 1 (COPY)", i);
        if (o.mode == 0) {
            if (it->second.children || it->second.requests)
                return fail(HALO_EBUSY, "send %d: MOVE of node %lld with %d children and %d requests", i,
                            (long long)o.node, it->second.children, it->second.requests);
            if (std::find(moved.begin(), moved.end(), o.node) != moved.end())
                return fail(HALO_EINVAL, "send %d: node %lld moved twice", i, (long long)o.node);
            moved.push_back(o.node);
        }
        if (o.peer == p->rank) self_send_tok.push_back(it->second.ntok);
    }
    for (int32_t i = 0; i < nrecv; ++i) {
        const auto &o = recvs[i];
        if (o.ntok < 1) return fail(HALO_EINVAL, "recv %d: ntok must be >= 1", i);
        if (o.peer < 0 || o.peer >= p->nranks) return fail(HALO_EINVAL, "recv %d: bad peer %d", i, o.peer);
        if (o.parent < -1) return fail(HALO_EINVAL, "recv %d: bad parent id", i);
        if (o.parent >= 0) {
            auto pit = p->nodes.find(o.parent);
            if (pit == p->nodes.end()) return fail(HALO_ENOENT, "recv %d: unknown parent %lld", i, (long long)o.parent);
            if (pit->second.on_host) return fail(HALO_EBUSY, "recv %d: parent %lld is offloaded", i, (long long)o.parent);
            if (std::find(moved.begin(), moved.end(), o.parent) != moved.end())
                return fail(HALO_EINVAL, "recv %d: parent %lld is moved away by this call", i, (long long)o.parent);
        }
        if (o.peer == p->rank) self_recv_tok.push_back(o.ntok);
    }
    if (self_send_tok != self_recv_tok)
        return fail(HALO_EINVAL, "self-loop sends and receives do not pair up (count or token counts differ)");
    DeviceGuard dg(p);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t run_bytes = (int64_t)p->cfg.num_kv_heads * kBlockTok * p->cfg.head_dim * 2;
    const int64_t item_bytes = 2 * run_bytes;  // K and V slab of one (layer, block)
    const int64_t R = std::max<int64_t>(1, p->mig_cfg.chunk_bytes / item_bytes);
    const int L = p->cfg.num_layers;
    // ---- destination blocks (all or nothing)
    std::vector<std::vector<int32_t>> dst(nrecv);
    for (int32_t i = 0; i < nrecv; ++i) {
        halo_status st = alloc_blocks(p, ceil_div(recvs[i].ntok, kBlockTok), dst[i]);
        if (st != HALO_OK) {
            for (int32_t j = i; j >= 0; --j) unalloc_blocks(p, dst[j], 0);
            return st;
        }
    }
    auto undo = [&]() {
        for (int32_t j = nrecv - 1; j >= 0; --j) unalloc_blocks(p, dst[j], 0);
    };
    // ---- transfers, buffer slices, block lists
    std::vector<Xfer> xs;
    std::vector<int32_t> lists;
    size_t per_parity = 0;
    int64_t rounds = 0;
    auto add = [&](bool snd, int32_t peer, const std::vector<int32_t> *blocks) {
        Xfer x;
        x.send = snd;
        x.peer = peer;
        x.nblk = (int64_t)blocks->size();
        x.items = x.nblk * L;
        x.nchunks = ceil_div(x.items, R);
        x.blocks = blocks;
        x.dev_off = (int64_t)lists.size();
        lists.insert(lists.end(), blocks->begin(), blocks->end());
        for (int32_t b : *blocks) lists.push_back((int32_t)p->blk_epoch[b]);  // V-table tags
        x.slice = (size_t)(std::min(R, x.items) * item_bytes);
        x.buf_off = per_parity;
        per_parity += x.slice;
        rounds = std::max(rounds, x.nchunks);
        xs.push_back(x);
    };
    for (int32_t i = 0; i < nsend; ++i) add(true, sends[i].peer, &p->nodes[sends[i].node].blocks);
    for (int32_t i = 0; i < nrecv; ++i) add(false, recvs[i].peer, &dst[i]);
    halo_status st = ensure_mig(p, 2 * per_parity);
    for (int32_t i = 0; i < nsend && st == HALO_OK; ++i) st = wait_ready(p, p->nodes[sends[i].node], s);
    Scratch sl;
    if (st == HALO_OK) st = upload(p, lists.data(), lists.size() * 4, s, sl);
    if (st != HALO_OK) {
        undo();
        return st;
    }
    // ---- rounds: pack(c) on s | one NCCL group of every transfer's chunk c on side | unpack(c-1)
    // on s.  Buffer reuse is ordered by construction: pack(c) follows unpack(c-2) on s, which
    // waited for round c-2; round c waits for pack(c).
    uint8_t *base = static_cast<uint8_t *>(p->mig_buf);
    cudaEvent_t *ev_packed = p->mig_ev, *ev_xfer = p->mig_ev + 2;
    const int32_t *dlist = static_cast<const int32_t *>(sl.ptr);
    const int ctas = p->mig_cfg.copy_ctas;
    auto unpack = [&](int64_t c) -> halo_status {
        const int b = (int)(c & 1);
        HALO_CUDA(cudaStreamWaitEvent(s, ev_xfer[b], 0));
        for (auto &x : xs) {
            if (x.send || c >= x.nchunks) continue;
            const int64_t i0 = c * R, i1 = std::min(x.items, i0 + R);
            cudaError_t e = launch_kv_runs(p->geom, p->k, p->v, base + b * per_parity + x.buf_off,
                                           dlist + x.dev_off, (const uint32_t *)(dlist + x.dev_off + x.nblk),
                                           (int32_t)x.nblk, i0, i1, true, ctas, s);
            if (e != cudaSuccess) return fail(HALO_ECUDA, "unpack launch: %s", cudaGetErrorString(e));
        }
        return HALO_OK;
    };
    // From the first launch on, an error leaves the exchange half-enqueued: the communicator
    // is unusable (peers wait), so it is reported as is.
    for (int64_t c = 0; c < rounds; ++c) {
        const int b = (int)(c & 1);
        for (auto &x : xs) {
            if (!x.send || c >= x.nchunks) continue;
            const int64_t i0 = c * R, i1 = std::min(x.items, i0 + R);
            cudaError_t e = launch_kv_runs(p->geom, p->k, p->v, base + b * per_parity + x.buf_off,
                                           dlist + x.dev_off, nullptr, (int32_t)x.nblk, i0, i1, false, ctas, s);
            if (e != cudaSuccess) return fail(HALO_ECUDA, "pack launch: %s", cudaGetErrorString(e));
        }
        HALO_CUDA(cudaEventRecord(ev_packed[b], s));
        HALO_CUDA(cudaStreamWaitEvent(p->side, ev_packed[b], 0));
        HALO_NCCL(nccl().GroupStart());
        for (auto &x : xs) {
            if (c >= x.nchunks) continue;
            const int64_t i0 = c * R, i1 = std::min(x.items, i0 + R);
            void *buf = base + b * per_parity + x.buf_off;
            const size_t bytes = (size_t)((i1 - i0) * item_bytes);
            ncclResult_t r = x.send ? nccl().Send(buf, bytes, ncclUint8, x.peer, p->comm, p->side)
                                    : nccl().Recv(buf, bytes, ncclUint8, x.peer, p->comm, p->side);
            if (r != ncclSuccess) {
                nccl().GroupEnd();
                return fail(HALO_ENCCL, "nccl %s of round %lld: %s", x.send ? "send" : "recv", (long long)c,
                            nccl().GetErrorString(r));
            }
        }
        HALO_NCCL(nccl().GroupEnd());
        HALO_CUDA(cudaEventRecord(ev_xfer[b], p->side));
        if (c > 0 && (st = unpack(c - 1)) != HALO_OK) return st;
    }
    if ((st = unpack(rounds - 1)) != HALO_OK) return st;  // also orders s after the last send
    HALO_CUDA(cudaEventRecord(p->mig_done, s));
    note_stream(p, s);
    // ---- bookkeeping: MOVE sources released (reusable once s has passed), receives registered
    for (int32_t i = 0; i < nsend; ++i) {
        if (sends[i].mode != 0) continue;
        auto it = p->nodes.find(sends[i].node);
        if (it == p->nodes.end()) continue;  // (listed twice as COPY and MOVE: already gone)
        const int64_t parent = it->second.parent;
        release_blocks(p, std::move(it->second.blocks));
        if (it->second.ready) p->event_cache.push_back(it->second.ready);
        p->nodes.erase(it);
        if (parent >= 0) p->nodes[parent].children--;
        p->layout_gen++;
    }
    for (int32_t i = 0; i < nrecv; ++i) {
        const int64_t id = p->next_id++;
        Node n;
        n.parent = recvs[i].parent;
        n.ntok = recvs[i].ntok;
        n.blocks = std::move(dst[i]);
        p->nodes.emplace(id, std::move(n));
        if (recvs[i].parent >= 0) p->nodes[recvs[i].parent].children++;
        nodes_out[i] = id;
    }
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_migrate_send(halo_pool p, int64_t node, int32_t dst_rank, int32_t mode, void *stream) {
    if (check_pool(p)) return HALO_EINVAL;
    if (dst_rank == p->rank) return fail(HALO_EINVAL, "send to self: use halo_migrate_exchange with the matching recv");
    halo_migrate_send_op o{node, dst_rank, mode};
    return halo_migrate_exchange(p, 1, &o, 0, nullptr, stream, nullptr);
}

halo_status halo_migrate_recv(halo_pool p, int32_t src_rank, int64_t parent, int32_t ntok, void *stream,
                              int64_t *node_out) {
    if (check_pool(p)) return HALO_EINVAL;
    if (src_rank == p->rank) return fail(HALO_EINVAL, "recv from self: use halo_migrate_exchange with the matching send");
    if (!node_out) return fail(HALO_EINVAL, "null node_out");
    halo_migrate_recv_op o{parent, src_rank, ntok};
    return halo_migrate_exchange(p, 0, nullptr, 1, &o, stream, node_out);
}

halo_status halo_prefix_clone(halo_pool src, int64_t node, halo_pool dst, int64_t parent_dst, void *stream,
                              int64_t *node_out) {
    HALO_GUARD_BEGIN
    if (check_pool(src) || check_pool(dst)) return HALO_EINVAL;
    if (src->host_only || dst->host_only) return fail(HALO_EUNSUPPORTED, "host-only pool");
    if (src->cfg.device != dst->cfg.device || src->cfg.num_layers != dst->cfg.num_layers ||
        src->cfg.num_kv_heads != dst->cfg.num_kv_heads || src->cfg.head_dim != dst->cfg.head_dim)
        return fail(HALO_EINVAL, "pools differ in device or KV geometry");
    auto it = src->nodes.find(node);
    if (it == src->nodes.end()) return fail(HALO_ENOENT, "unknown node %lld", (long long)node);
    if (it->second.on_host) return fail(HALO_EBUSY, "node %lld is offloaded: fetch it first", (long long)node);
    if (!node_out) return fail(HALO_EINVAL, "null node_out");
    if (parent_dst >= 0 && !dst->nodes.count(parent_dst))
        return fail(HALO_ENOENT, "unknown parent %lld", (long long)parent_dst);
    DeviceGuard dg(src);
    cudaStream_t s = (cudaStream_t)stream;
    halo_status st = wait_ready(src, it->second, s);
    if (st != HALO_OK) return st;
    const int32_t ntok = it->second.ntok;
    const int64_t nblk = ceil_div(ntok, kBlockTok);
    std::vector<int32_t> blocks;
    st = alloc_blocks(dst, nblk, blocks);
    if (st != HALO_OK) return st;
    // whole-block pool-to-pool copy: a (layer, block) of all heads is contiguous on both sides
    std::vector<int32_t> pairs(3 * nblk);  // pairs | destination tags
    for (int64_t b = 0; b < nblk; ++b) {
        pairs[2 * b] = it->second.blocks[b];
        pairs[2 * b + 1] = blocks[b];
        pairs[2 * nblk + b] = (int32_t)dst->blk_epoch[blocks[b]];
    }
    Scratch sp;
    if ((st = upload(src, pairs.data(), pairs.size() * 4, s, sp)) == HALO_OK) {
        const int32_t *dp = (const int32_t *)sp.ptr;
        cudaError_t e = launch_kv_copy_blocks(src->geom, src->k, src->v, dst->geom, dst->k, dst->v, dp,
                                              (const uint32_t *)(dp + 2 * nblk), (int32_t)nblk, 0,
                                              src->cfg.num_layers, src->num_sms, s);
        if (e != cudaSuccess) st = fail(HALO_ECUDA, "clone launch: %s", cudaGetErrorString(e));
    }
    if (st != HALO_OK) {
        unalloc_blocks(dst, blocks, 0);
        return st;
    }
    note_stream(src, s);
    note_stream(dst, s);
    const int64_t id = dst->next_id++;
    Node n;
    n.parent = parent_dst;
    n.ntok = ntok;
    n.blocks = std::move(blocks);
    dst->nodes.emplace(id, std::move(n));
    if (parent_dst >= 0) dst->nodes[parent_dst].children++;
    *node_out = id;
    return HALO_OK;
    HALO_GUARD_END
}

// ---------------------------------------------------------------- host paging API
halo_status halo_pool_host_reserve(halo_pool p, int64_t host_blocks) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    if (host_blocks < 0 || host_blocks * p->cfg.num_kv_heads > (int64_t)kBlkMask + 1 ||
        (int64_t)p->cfg.num_layers * host_blocks >= ((int64_t)1 << 31))
        return fail(HALO_EINVAL, "host_blocks out of range");
    for (auto &n : p->nodes)
        if (n.second.on_host) return fail(HALO_EBUSY, "nodes are offloaded to the current arena");
    DeviceGuard dg(p);
    if (!p->host_only) {
        for (auto &pf : p->host_pending)
            for (cudaEvent_t e : pf.events) cudaEventSynchronize(e);
        if (p->hk) cudaFreeHost(p->hk);
        if (p->hv) cudaFreeHost(p->hv);
        p->hk = p->hv = nullptr;
        const size_t bytes = (size_t)p->cfg.num_layers * host_blocks * p->cfg.num_kv_heads * kBlockTok *
                             p->cfg.head_dim * 2;
        if (bytes && (cudaHostAlloc(&p->hk, bytes, cudaHostAllocDefault) != cudaSuccess ||
                      cudaHostAlloc(&p->hv, bytes, cudaHostAllocDefault) != cudaSuccess)) {
            cudaGetLastError();
            if (p->hk) cudaFreeHost(p->hk);
            p->hk = p->hv = nullptr;
            p->host_cap = 0;
            p->host_free.clear();
            return fail(HALO_ENOMEM, "pinned host arena of %zu bytes x 2", bytes);
        }
    }
    for (auto &pf : p->host_pending) p->event_cache.insert(p->event_cache.end(), pf.events.begin(), pf.events.end());
    p->host_pending.clear();
    p->host_cap = host_blocks;
    p->host_free.clear();
    for (int64_t b = host_blocks - 1; b >= 0; --b) p->host_free.push_back((int32_t)b);
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_prefix_offload(halo_pool p, int64_t node, void *stream) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    auto it = p->nodes.find(node);
    if (it == p->nodes.end()) return fail(HALO_ENOENT, "unknown node %lld", (long long)node);
    if (it->second.on_host) return fail(HALO_EINVAL, "node %lld is already offloaded", (long long)node);
    if (p->host_cap == 0) return fail(HALO_EUNSUPPORTED, "no host arena (halo_pool_host_reserve)");
    DeviceGuard dg(p);
    return offload_node(p, it->second, (cudaStream_t)stream);
    HALO_GUARD_END
}

halo_status halo_prefix_fetch(halo_pool p, int64_t node, void *stream) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    auto it = p->nodes.find(node);
    if (it == p->nodes.end()) return fail(HALO_ENOENT, "unknown node %lld", (long long)node);
    Node &n = it->second;
    if (!n.on_host) return fail(HALO_EINVAL, "node %lld is not offloaded", (long long)node);
    DeviceGuard dg(p);
    std::vector<int32_t> db;
    halo_status st = alloc_blocks(p, (int64_t)n.host_blocks.size(), db);
    if (st != HALO_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if (!p->host_only) {
        std::vector<int32_t> bt(db);  // blocks | tags: the V-table entries are recomputed
        for (int32_t b : db) bt.push_back((int32_t)p->blk_epoch[b]);
        Scratch sb;
        st = upload(p, bt.data(), bt.size() * 4, s, sb);
        if (st == HALO_OK) st = copy_node_blocks(p, db, n.host_blocks, false, s);
        if (st == HALO_OK) {
            const int32_t *d = (const int32_t *)sb.ptr;
            cudaError_t e = launch_kv_vmax(p->geom, p->v, d, (const uint32_t *)(d + db.size()), (int32_t)db.size(),
                                           p->num_sms, s);
            if (e != cudaSuccess) st = fail(HALO_ECUDA, "V-table launch: %s", cudaGetErrorString(e));
        }
        if (st == HALO_OK) {
            if (!n.ready) n.ready = get_event(p);
            if (!n.ready || cudaEventRecord(n.ready, s) != cudaSuccess)
                st = fail(HALO_ECUDA, "fetch event record failed");
        }
        if (st != HALO_OK) {
            unalloc_blocks(p, db, 0);
            return st;
        }
        note_stream(p, s);
    }
    release_host_blocks(p, std::move(n.host_blocks));  // reusable once the copy has passed
    n.host_blocks.clear();
    n.blocks = std::move(db);
    n.on_host = false;
    // (no plan can reference an offloaded node -- building one fails with EBUSY -- so a fetch
    // leaves existing plans valid: a step's plan keeps running while the next step prefetches)
    return HALO_OK;
    HALO_GUARD_END
}

halo_status halo_pool_prefetch(halo_pool p, int32_t nreq, const int64_t *reqs, void *stream, int32_t *n_fetched) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    if (nreq < 0 || (nreq > 0 && !reqs)) return fail(HALO_EINVAL, "bad request list");
    std::vector<int64_t> want;  // offloaded nodes on the requests' paths, parents first
    for (int32_t i = 0; i < nreq; ++i) {
        auto r = p->requests.find(reqs[i]);
        if (r == p->requests.end()) return fail(HALO_ENOENT, "unknown request %lld", (long long)reqs[i]);
        std::vector<int64_t> path;
        for (int64_t id = r->second.leaf; id >= 0; id = p->nodes[id].parent) path.push_back(id);
        for (auto it = path.rbegin(); it != path.rend(); ++it)
            if (p->nodes[*it].on_host && std::find(want.begin(), want.end(), *it) == want.end()) want.push_back(*it);
    }
    int32_t n = 0;
    halo_status st = HALO_OK;
    for (int64_t id : want) {
        if ((st = halo_prefix_fetch(p, id, stream)) != HALO_OK) break;
        ++n;
    }
    if (n_fetched) *n_fetched = n;
    return st;
    HALO_GUARD_END
}

halo_status halo_node_residency(halo_pool p, int64_t node, int32_t *on_device, uint64_t *last_use) {
    if (check_pool(p)) return HALO_EINVAL;
    auto it = p->nodes.find(node);
    if (it == p->nodes.end()) return fail(HALO_ENOENT, "unknown node %lld", (long long)node);
    if (on_device) *on_device = it->second.on_host ? 0 : 1;
    if (last_use) *last_use = it->second.last_use;
    return HALO_OK;
}

halo_status halo_pool_evict_lru(halo_pool p, int64_t want_free, void *stream, int32_t *n_evicted) {
    HALO_GUARD_BEGIN
    if (check_pool(p)) return HALO_EINVAL;
    if (p->host_cap == 0) return fail(HALO_EUNSUPPORTED, "no host arena (halo_pool_host_reserve)");
    DeviceGuard dg(p);
    auto free_now = [&]() {
        int64_t f = (int64_t)p->free_list.size();
        for (auto &pf : p->pending) f += (int64_t)pf.blocks.size();
        return f;
    };
    // candidates: device-resident nodes not read by the latest plan, least recently used
    // first (ties: lower id)
    std::vector<std::pair<uint64_t, int64_t>> cand;
    for (auto &n : p->nodes)
        if (!n.second.on_host && !n.second.blocks.empty() && n.second.last_use < p->plan_tick)
            cand.push_back({n.second.last_use, n.first});
    std::sort(cand.begin(), cand.end());
    int32_t ev = 0;
    for (auto &c : cand) {
        if (free_now() >= want_free) break;
        Node &n = p->nodes[c.second];
        if ((int64_t)p->host_free.size() < (int64_t)n.blocks.size()) reclaim_host(p, false);
        if ((int64_t)p->host_free.size() < (int64_t)n.blocks.size()) break;  // arena full
        halo_status st = offload_node(p, n, (cudaStream_t)stream);
        if (st != HALO_OK) return st;
        ++ev;
    }
    if (n_evicted) *n_evicted = ev;
    if (free_now() < want_free)
        return fail(HALO_ENOMEM, "could not free %lld blocks by eviction", (long long)want_free);
    return HALO_OK;
    HALO_GUARD_END
}

}  // extern "C"
