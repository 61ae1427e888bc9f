"""ctypes binding of include/halo_attn.h (same names as the C ABI, Pythonic wrappers).

Marshalling only: tensors are passed as raw pointers, streams as cudaStream_t handles.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_PKG, "libhalo_attn.so")

STATUS = {0: "HALO_OK", 1: "HALO_EINVAL", 2: "HALO_ENOMEM", 3: "HALO_ENOENT", 4: "HALO_EBUSY",
          5: "HALO_ECUDA", 6: "HALO_ENCCL", 7: "HALO_EUNSUPPORTED"}

# Every symbol include/halo_attn.h declares, with its ctypes signature.
_i32, _i64, _p, _f = C.c_int32, C.c_int64, C.c_void_p, C.c_float
_pi64, _pi32 = C.POINTER(C.c_int64), C.POINTER(C.c_int32)


class PoolConfig(C.Structure):
    _fields_ = [("device", _i32), ("num_layers", _i32), ("num_kv_heads", _i32),
                ("num_q_heads", _i32), ("head_dim", _i32), ("block_tokens", _i32),
                ("capacity_blocks", _i64), ("k_storage", _p), ("v_storage", _p)]


class PlanOptions(C.Structure):
    _fields_ = [("min_tensor_rows", _i32), ("force_splits", _i32), ("max_splits", _i32),
                ("k2_chunk_blocks", _i32), ("k2_shape", _i32), ("k2_sms", _i32),
                ("k1_sm_frac", C.c_float), ("k2_early_weight", C.c_float),
                ("k2_tail_pct", _i32), ("k2_whole_units", _i32)]


class PlanInfo(C.Structure):
    _fields_ = [("nreq", _i32), ("num_q_heads", _i32), ("num_kv_heads", _i32), ("head_dim", _i32),
                ("tensor_nodes", _i32), ("folded_nodes", _i32), ("k1_tiles", _i32),
                ("k2_units", _i32), ("max_slots", _i32), ("k2_warps", _i32), ("k1_rows", _i64),
                ("k1_flops", C.c_double), ("k1_bytes", C.c_double), ("k2_bytes", C.c_double),
                ("unshared_bytes", C.c_double)]


class PlaceItem(C.Structure):
    _fields_ = [("exec_s", C.c_double), ("kv_bytes", C.c_double), ("prep_s", C.c_double),
                ("home", _i32), ("max_replicas", _i32)]


class PlaceConfig(C.Structure):
    _fields_ = [("workers", _i32), ("beam_width", _i32), ("ops_per_iter", _i32), ("reserved", _i32),
                ("beta", C.c_double), ("link_bytes_per_s", C.c_double)]


class PlaceMove(C.Structure):
    _fields_ = [("item", _i32), ("src", _i32), ("dst", _i32), ("mode", _i32), ("seconds", C.c_double)]


class CommConfig(C.Structure):
    _fields_ = [("max_ctas", _i32), ("copy_ctas", _i32), ("chunk_bytes", _i64)]


class MigrateSendOp(C.Structure):
    _fields_ = [("node", _i64), ("peer", _i32), ("mode", _i32)]


class MigrateRecvOp(C.Structure):
    _fields_ = [("parent", _i64), ("peer", _i32), ("ntok", _i32)]


SIGNATURES = {
    "halo_last_error": (C.c_char_p, []),
    "halo_abi_version": (_i32, []),
    "halo_pool_storage_bytes": (C.c_size_t, [C.POINTER(PoolConfig)]),
    "halo_pool_create": (_i32, [C.POINTER(PoolConfig), C.POINTER(_p)]),
    "halo_pool_destroy": (_i32, [_p]),
    "halo_pool_stats": (_i32, [_p, _pi64, _pi64]),
    "halo_pool_storage": (_i32, [_p, C.POINTER(_p), C.POINTER(_p)]),
    "halo_prefix_register": (_i32, [_p, _i64, _i32, _p, _p, _p, _pi64]),
    "halo_prefix_release": (_i32, [_p, _i64]),
    "halo_prefix_read": (_i32, [_p, _i64, _p, _p, _p]),
    "halo_node_info": (_i32, [_p, _i64, _pi64, _pi32, _pi32, _pi32]),
    "halo_request_open": (_i32, [_p, _i64, _pi64]),
    "halo_request_close": (_i32, [_p, _i64]),
    "halo_request_info": (_i32, [_p, _i64, _pi64, _pi32, _pi32]),
    "halo_suffix_append": (_i32, [_p, _i32, _pi64, _pi32, _p, _p, _p]),
    "halo_suffix_truncate": (_i32, [_p, _i32, _pi64, _pi32]),
    "halo_decode_plan": (_i32, [_p, _i32, _pi64, C.POINTER(PlanOptions), _p, C.POINTER(_p)]),
    "halo_decode_run": (_i32, [_p, _i32, _p, _p, _p, _f, _p]),
    "halo_decode_run_stages": (_i32, [_p, _i32, _i32, _p, _p, _p, _f, _p]),
    "halo_decode_layers": (_i32, [_p, _i32, _p, _p, _p, _f, _p]),
    "halo_prefill_plan": (_i32, [_p, _i32, _pi64, _pi32, C.POINTER(PlanOptions), _p, C.POINTER(_p)]),
    "halo_decode_step": (_i32, [_p, _i32, _pi64, _p, _p, _p, _p, _p, _f, C.POINTER(PlanOptions), _p,
                                C.POINTER(_p)]),
    "halo_plan_get_info": (_i32, [_p, C.POINTER(PlanInfo)]),
    "halo_plan_export": (_i32, [_p, _i32, _p, _i64, _pi64]),
    "halo_plan_destroy": (_i32, [_p]),
    "halo_comm_unique_id": (_i32, [_p]),
    "halo_comm_init": (_i32, [_p, _p, _i32, _i32]),
    "halo_comm_init_config": (_i32, [_p, _p, _i32, _i32, C.POINTER(CommConfig)]),
    "halo_migrate_exchange": (_i32, [_p, _i32, C.POINTER(MigrateSendOp), _i32, C.POINTER(MigrateRecvOp),
                                     _p, _pi64]),
    "halo_migrate_send": (_i32, [_p, _i64, _i32, _i32, _p]),
    "halo_migrate_recv": (_i32, [_p, _i32, _i64, _i32, _p, _pi64]),
    "halo_prefix_clone": (_i32, [_p, _i64, _p, _i64, _p, _pi64]),
    "halo_pool_host_reserve": (_i32, [_p, _i64]),
    "halo_prefix_offload": (_i32, [_p, _i64, _p]),
    "halo_prefix_fetch": (_i32, [_p, _i64, _p]),
    "halo_node_residency": (_i32, [_p, _i64, C.POINTER(C.c_int32), C.POINTER(C.c_uint64)]),
    "halo_pool_prefetch": (_i32, [_p, _i32, _pi64, _p, C.POINTER(C.c_int32)]),
    "halo_pool_evict_lru": (_i32, [_p, _i64, _p, C.POINTER(C.c_int32)]),
    "halo_place_groups": (_i32, [C.POINTER(PlaceConfig), _i32, C.POINTER(PlaceItem),
                                 C.POINTER(C.c_uint64), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                 C.POINTER(PlaceMove), _i32, C.POINTER(C.c_int32)]),
}

_lib = None


def lib_path() -> str:
    # HALO_LIB selects a debug build of the same library (e.g. libhalo_attn_trace.so)
    return os.environ.get("HALO_LIB", _LIB_PATH)


def load_library():
    """Load libhalo_attn.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: build it with "
                              "`python -m paper_2509_02121_b200.build` (no CPU fallback exists)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            if "HALO_LIB" in os.environ and not hasattr(lib, name):
                continue  # a debug / A-B build of another revision: bind what it has
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class HaloError(RuntimeError):
    def __init__(self, status: int, fn: str, msg: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{fn}: {self.name}: {msg}")


def _check(fn: str, st: int):
    if st != 0:
        msg = load_library().halo_last_error().decode(errors="replace")
        raise HaloError(st, fn, msg)


def _call(fn: str, *args):
    _check(fn, getattr(load_library(), fn)(*args))


def _ptr(t) -> int | None:
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        assert t.is_contiguous(), "tensors crossing the ABI must be contiguous"
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        assert t.flags["C_CONTIGUOUS"]
        return t.ctypes.data
    return int(t)


def _stream(stream, device: int):
    if stream is not None:
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    if device < 0:
        return None
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def _i64_array(xs):
    a = (C.c_int64 * len(xs))(*[int(x) for x in xs])
    return a


def _i32_array(xs):
    return (C.c_int32 * len(xs))(*[int(x) for x in xs])


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _call("halo_comm_unique_id", buf)
    return buf.raw


def place_groups(items, workers: int, beam_width: int = 16, ops_per_iter: int = 1,
                 beta: float = 1.0, link_bytes_per_s: float = 1e11) -> dict:
    """halo_place_groups: the relocation planner (Alg. 1 with the §3.2 costs).
    items: sequence of dicts with exec_s, kv_bytes, prep_s (default 0), home (default -1),
    max_replicas (default 1).  Returns {"workers": [list of worker indices per item],
    "masks", "load", "cost", "moves": [(item, src, dst, mode, seconds)]}."""
    n = len(items)
    arr = (PlaceItem * max(n, 1))()
    for i, it in enumerate(items):
        arr[i] = PlaceItem(float(it["exec_s"]), float(it.get("kv_bytes", 0.0)),
                           float(it.get("prep_s", 0.0)), int(it.get("home", -1)),
                           int(it.get("max_replicas", 1)))
    cfg = PlaceConfig(int(workers), int(beam_width), int(ops_per_iter), 0, float(beta),
                      float(link_bytes_per_s))
    masks = (C.c_uint64 * max(n, 1))()
    load = (C.c_double * max(int(workers), 1))()
    cost = C.c_double(0.0)
    cap = max(n * max(int(workers), 1), 1)
    moves = (PlaceMove * cap)()
    nm = C.c_int32(0)
    _call("halo_place_groups", C.byref(cfg), n, arr, masks, load, C.byref(cost), moves, cap,
          C.byref(nm))
    ms = [int(masks[i]) for i in range(n)]
    return {"masks": ms,
            "workers": [[d for d in range(workers) if m >> d & 1] for m in ms],
            "load": [load[d] for d in range(workers)],
            "cost": cost.value,
            "moves": [(moves[i].item, moves[i].src, moves[i].dst, moves[i].mode, moves[i].seconds)
                      for i in range(nm.value)]}


class Pool:
    """A paged bf16 KV pool [layer][block][kv_head][16][d] (halo_pool_create)."""

    def __init__(self, num_layers: int, num_kv_heads: int, num_q_heads: int, head_dim: int,
                 capacity_blocks: int, device: int = 0, k_storage=None, v_storage=None):
        self.cfg = PoolConfig(device, num_layers, num_kv_heads, num_q_heads, head_dim, 16,
                              capacity_blocks, _ptr(k_storage), _ptr(v_storage))
        self.device = device
        self._keep = (k_storage, v_storage)
        h = C.c_void_p()
        _call("halo_pool_create", C.byref(self.cfg), C.byref(h))
        self.handle = h

    @property
    def layers(self):
        return self.cfg.num_layers

    @property
    def hkv(self):
        return self.cfg.num_kv_heads

    @property
    def hq(self):
        return self.cfg.num_q_heads

    @property
    def d(self):
        return self.cfg.head_dim

    def storage_bytes(self) -> int:
        return load_library().halo_pool_storage_bytes(C.byref(self.cfg))

    def destroy(self):
        if self.handle:
            _call("halo_pool_destroy", self.handle)
            self.handle = None

    def stats(self):
        f, u = C.c_int64(), C.c_int64()
        _call("halo_pool_stats", self.handle, C.byref(f), C.byref(u))
        return f.value, u.value

    def storage(self):
        k, v = C.c_void_p(), C.c_void_p()
        _call("halo_pool_storage", self.handle, C.byref(k), C.byref(v))
        return k.value, v.value

    def _s(self, stream):
        return _stream(stream, self.device)

    def register_prefix(self, parent: int, ntok: int, k=None, v=None, stream=None) -> int:
        out = C.c_int64()
        _call("halo_prefix_register", self.handle, parent, ntok, _ptr(k), _ptr(v),
              self._s(stream), C.byref(out))
        return out.value

    def release_prefix(self, node: int):
        _call("halo_prefix_release", self.handle, node)

    def read_prefix(self, node: int, k_out, v_out, stream=None):
        _call("halo_prefix_read", self.handle, node, _ptr(k_out), _ptr(v_out), self._s(stream))

    def node_info(self, node: int) -> dict:
        parent, ntok, nb = C.c_int64(), C.c_int32(), C.c_int32()
        _call("halo_node_info", self.handle, node, C.byref(parent), C.byref(ntok), C.byref(nb), None)
        blocks = (C.c_int32 * max(nb.value, 1))()
        _call("halo_node_info", self.handle, node, None, None, None, blocks)
        return {"parent": parent.value, "ntok": ntok.value,
                "blocks": list(blocks)[:nb.value]}

    def open_request(self, leaf: int = -1) -> int:
        out = C.c_int64()
        _call("halo_request_open", self.handle, leaf, C.byref(out))
        return out.value

    def close_request(self, req: int):
        _call("halo_request_close", self.handle, req)

    def request_info(self, req: int) -> dict:
        leaf, ln, nb = C.c_int64(), C.c_int32(), C.c_int32()
        _call("halo_request_info", self.handle, req, C.byref(leaf), C.byref(ln), C.byref(nb))
        return {"leaf": leaf.value, "suffix_len": ln.value, "nblocks": nb.value}

    def append(self, reqs, ntok, k=None, v=None, stream=None):
        _call("halo_suffix_append", self.handle, len(reqs), _i64_array(reqs), _i32_array(ntok),
              _ptr(k), _ptr(v), self._s(stream))

    def truncate(self, reqs, ntok):
        _call("halo_suffix_truncate", self.handle, len(reqs), _i64_array(reqs), _i32_array(ntok))

    def plan(self, reqs, options: PlanOptions | None = None, stream=None, reuse: "Plan" = None):
        h = C.c_void_p(reuse.handle.value if reuse is not None else None)
        _call("halo_decode_plan", self.handle, len(reqs), _i64_array(reqs),
              C.byref(options) if options is not None else None, self._s(stream), C.byref(h))
        if reuse is not None:
            reuse.nreq = len(reqs)
            return reuse
        return Plan(self, h, len(reqs))

    def prefill_plan(self, reqs, ntok, options: PlanOptions | None = None, stream=None,
                     reuse: "Plan" = None):
        """halo_prefill_plan: rows = the last ntok[i] suffix tokens of each request (causal)."""
        h = C.c_void_p(reuse.handle.value if reuse is not None else None)
        _call("halo_prefill_plan", self.handle, len(reqs), _i64_array(reqs), _i32_array(ntok),
              C.byref(options) if options is not None else None, self._s(stream), C.byref(h))
        rows = int(sum(ntok))
        if reuse is not None:
            reuse.nreq = rows
            return reuse
        return Plan(self, h, rows)

    def decode_step(self, reqs, k_new, v_new, q, out, lse=None, scale: float = 0.0,
                    options: PlanOptions | None = None, stream=None, reuse: "Plan" = None):
        """halo_decode_step: append one token per request, (re)plan, attend every layer,
        with per-layer overlap of host<->device copies (host tensors should be pinned)."""
        h = C.c_void_p(reuse.handle.value if reuse is not None else None)
        _call("halo_decode_step", self.handle, len(reqs), _i64_array(reqs), _ptr(k_new), _ptr(v_new),
              _ptr(q), _ptr(out), _ptr(lse), scale, C.byref(options) if options is not None else None,
              self._s(stream), C.byref(h))
        if reuse is not None:
            reuse.nreq = len(reqs)
            return reuse
        return Plan(self, h, len(reqs))

    # ---- host paging ----
    def host_reserve(self, host_blocks: int):
        _call("halo_pool_host_reserve", self.handle, host_blocks)

    def offload_prefix(self, node: int, stream=None):
        _call("halo_prefix_offload", self.handle, node, self._s(stream))

    def fetch_prefix(self, node: int, stream=None):
        _call("halo_prefix_fetch", self.handle, node, self._s(stream))

    def prefetch(self, reqs, stream=None) -> int:
        n = C.c_int32()
        _call("halo_pool_prefetch", self.handle, len(reqs), _i64_array(reqs), self._s(stream), C.byref(n))
        return int(n.value)

    def residency(self, node: int) -> tuple:
        on, last = C.c_int32(), C.c_uint64()
        _call("halo_node_residency", self.handle, node, C.byref(on), C.byref(last))
        return bool(on.value), int(last.value)

    def evict_lru(self, want_free: int, stream=None) -> int:
        n = C.c_int32()
        _call("halo_pool_evict_lru", self.handle, want_free, self._s(stream), C.byref(n))
        return int(n.value)

    # ---- migration ----
    def comm_init(self, uid: bytes, nranks: int, rank: int, max_ctas: int = 0, copy_ctas: int = 0,
                  chunk_bytes: int = 0):
        buf = C.create_string_buffer(uid, 128)
        if max_ctas or copy_ctas or chunk_bytes:
            cfg = CommConfig(max_ctas, copy_ctas, chunk_bytes)
            _call("halo_comm_init_config", self.handle, buf, nranks, rank, C.byref(cfg))
        else:
            _call("halo_comm_init", self.handle, buf, nranks, rank)

    def migrate_exchange(self, sends=(), recvs=(), stream=None) -> list:
        """sends: [(node, peer, mode)], recvs: [(peer, parent, ntok)] -> new node ids (recv order)."""
        ns, nr = len(sends), len(recvs)
        sa = (MigrateSendOp * max(ns, 1))(*[MigrateSendOp(n, pr, m) for n, pr, m in sends])
        ra = (MigrateRecvOp * max(nr, 1))(*[MigrateRecvOp(par, pr, nt) for pr, par, nt in recvs])
        out = (C.c_int64 * max(nr, 1))()
        _call("halo_migrate_exchange", self.handle, ns, sa, nr, ra, self._s(stream), out)
        return [int(out[i]) for i in range(nr)]

    def migrate_send(self, node: int, dst_rank: int, mode: int = 1, stream=None):
        _call("halo_migrate_send", self.handle, node, dst_rank, mode, self._s(stream))

    def migrate_recv(self, src_rank: int, parent: int, ntok: int, stream=None) -> int:
        out = C.c_int64()
        _call("halo_migrate_recv", self.handle, src_rank, parent, ntok, self._s(stream),
              C.byref(out))
        return out.value

    def clone_prefix(self, node: int, dst: "Pool", parent: int = -1, stream=None) -> int:
        out = C.c_int64()
        _call("halo_prefix_clone", self.handle, node, dst.handle, parent, self._s(stream),
              C.byref(out))
        return out.value


EXPORTS = {"req_order": 0, "tiles": 1, "req_nslots": 2, "unit_req": 3, "req_blk_off": 4,
           "req_blk": 5, "unit_boff": 6, "chunk_u0": 7, "chunk_u1": 8, "unit_nseg": 9,
           "chunk_lo": 10}


class Plan:
    """One decode step's plan (halo_decode_plan); run it per layer (halo_decode_run)."""

    def __init__(self, pool: Pool, handle, nreq: int):
        self.pool, self.handle, self.nreq = pool, handle, nreq

    def run(self, layer: int, q, out, lse=None, scale: float = 0.0, stream=None):
        _call("halo_decode_run", self.handle, layer, _ptr(q), _ptr(out), _ptr(lse), scale,
              self.pool._s(stream))

    def run_stages(self, layer: int, mask: int, q, out=None, lse=None, scale: float = 0.0,
                   stream=None):
        _call("halo_decode_run_stages", self.handle, layer, mask, _ptr(q), _ptr(out), _ptr(lse),
              scale, self.pool._s(stream))

    def run_layers(self, nlayers: int, q, out, lse=None, scale: float = 0.0, stream=None):
        _call("halo_decode_layers", self.handle, nlayers, _ptr(q), _ptr(out), _ptr(lse), scale,
              self.pool._s(stream))

    def info(self) -> dict:
        inf = PlanInfo()
        _call("halo_plan_get_info", self.handle, C.byref(inf))
        return {name: getattr(inf, name) for name, _ in PlanInfo._fields_}

    def export(self, which: str) -> np.ndarray:
        code = EXPORTS[which]
        n = C.c_int64()
        _call("halo_plan_export", self.handle, code, None, 0, C.byref(n))
        dt = np.uint32 if which == "req_blk" else np.int32
        arr = np.zeros(max(n.value, 1), dtype=dt)
        _call("halo_plan_export", self.handle, code, arr.ctypes.data, n.value, C.byref(n))
        arr = arr[:n.value]
        return arr.reshape(-1, 8) if which == "tiles" else arr

    def destroy(self):
        if self.handle:
            _call("halo_plan_destroy", self.handle)
            self.handle = None
