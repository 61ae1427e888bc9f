"""Populate a Pool from a synthetic workload spec (synth.Workload) through the public API.

Glue for tests, smoke() and bench.py: it only calls halo_prefix_register /
halo_request_open / halo_suffix_append with tensors produced by the seeded generator.
"""
from __future__ import annotations

from dataclasses import dataclass

from .abi import Pool


def blocks_needed(wl, steps: int = 1, slack: int = 64) -> int:
    n = sum((nd.ntok + 15) // 16 for nd in wl.nodes)
    n += sum((r.suffix + steps + 15) // 16 for r in wl.requests)
    return n + slack


@dataclass
class Loaded:
    pool: Pool
    node_ids: dict   # workload node ident -> pool node id
    req_ids: list    # workload request index -> pool request id


def load(wl, device: int = 0, capacity: int | None = None, stream=None, pool: Pool | None = None,
         gen_device=None) -> Loaded:
    """Register every prefix node (parents first), open the requests, append the initial
    suffixes.  Tensors are generated on `gen_device` (default: the pool's GPU)."""
    import torch
    dev = gen_device if gen_device is not None else (f"cuda:{device}" if device >= 0 else "cpu")
    if pool is None:
        pool = Pool(wl.layers, wl.hkv, wl.hq, wl.d, capacity or blocks_needed(wl), device)
    depth = {}

    def dep(n):
        if n not in depth:
            p = wl.node(n).parent
            depth[n] = 0 if p < 0 else dep(p) + 1
        return depth[n]

    node_ids = {}
    for nd in sorted(wl.nodes, key=lambda x: (dep(x.ident), x.ident)):
        k = v = None
        if device >= 0:
            k, v = wl.node_kv(nd.ident, dev)
        parent = node_ids[nd.parent] if nd.parent >= 0 else -1
        node_ids[nd.ident] = pool.register_prefix(parent, nd.ntok, k, v, stream)
        del k, v
    req_ids = [pool.open_request(node_ids[r.leaf] if r.leaf >= 0 else -1) for r in wl.requests]
    if int(wl.suffix_offsets[-1]) > 0:
        k = v = None
        if device >= 0:
            k, v = wl.suffix_kv(dev)
        pool.append(req_ids, [r.suffix for r in wl.requests], k, v, stream)
        del k, v
        if device >= 0:
            torch.cuda.synchronize(device)
    return Loaded(pool, node_ids, req_ids)


def append_step(ld: Loaded, wl, step: int, device: int = 0, stream=None):
    """Append the token of decode step `step` (one per request, all layers)."""
    k = v = None
    if device >= 0:
        k, v = wl.new_kv(step, f"cuda:{device}")
    ld.pool.append(ld.req_ids, [1] * len(ld.req_ids), k, v, stream)
    return k, v
