"""Cost-model-driven relocation: decide where each prefix group's
KV should live with the library's planner (halo_place_groups: PAPER.md Alg. 1 beam search
with the §3.2 cost functions), then move the KV with the
migration path -- "cache snapshots ... migrated among GPUs via NVLink ... under scheduler
control".

Host glue only (marshalling and bookkeeping).  The planner is native (placement.cpp); the
KV moves are the library's clone / NCCL send-recv kernels.

* `group_items`   -- one planner item per prefix group (sharding.subtree_groups): e_v from
                     the two rooflines (K1 FLOPs / tensor rate + K2 bytes / HBM rate) over
                     the decode horizon, kv_bytes of the group's prefix nodes, p_v for a group
                     no worker holds = a host fetch at the measured PCIe rate.
* `rank_actions`  -- the per-rank send / recv / prepare sequence of a move list.  Every rank
                     walks the moves in the planner's global order, so each pair's sends and
                     receives match in order and the transfers cannot deadlock (the partner of
                     a blocked transfer is always at an earlier or the same global index).
* `execute_local` -- realise a placement between pools of one process (workers = pools on
                     one GPU): halo_prefix_clone of each node of the group (parents first),
                     then release of the source subtree on MOVE.
"""
from __future__ import annotations

from .abi import place_groups
from .sharding import DEFAULT_HBM_BPS, DEFAULT_TC_FLOPS, subtree_groups


def group_items(wl, homes, steps: int = 1, tc_flops: float = DEFAULT_TC_FLOPS,
                hbm_bps: float = DEFAULT_HBM_BPS, fetch_bytes_per_s: float = 5e10,
                max_replicas: int = 1, min_rows: int = 64):
    """(groups, items): one item per prefix group of `wl`.  homes[i] = worker holding group
    i's KV now (-1: none, i.e. offloaded to the host arena).  exec_s = per-layer roofline
    cost x layers x steps; kv_bytes = the group's prefix tokens x layers x K+V bytes."""
    groups = subtree_groups(wl, tc_flops=tc_flops, hbm_bps=hbm_bps, min_rows=min_rows)
    if len(homes) != len(groups):
        raise ValueError(f"{len(homes)} homes for {len(groups)} groups")
    ntok = {nd.ident: nd.ntok for nd in wl.nodes}
    kv_tok = wl.hkv * wl.d * 2 * 2 * wl.layers
    items = []
    for g, h in zip(groups, homes):
        kvb = float(sum(ntok[n] for n in g.nodes) * kv_tok)
        items.append({"exec_s": g.cost * wl.layers * steps, "kv_bytes": kvb,
                      "prep_s": kvb / fetch_bytes_per_s, "home": int(h),
                      "max_replicas": max_replicas if g.root >= 0 else 1})
    return groups, items


def plan_relocation(wl, homes, workers: int, link_bytes_per_s: float, beam_width: int = 16,
                    ops_per_iter: int = 1, beta: float = 1.0, **kw):
    """Run the planner on `wl`'s prefix groups.  Returns (groups, items, placement dict)."""
    groups, items = group_items(wl, homes, **kw)
    res = place_groups(items, workers, beam_width=beam_width, ops_per_iter=ops_per_iter,
                       beta=beta, link_bytes_per_s=link_bytes_per_s)
    return groups, items, res


def rank_actions(moves, rank: int):
    """This rank's part of a move list, in global order: ("send", item, dst, mode),
    ("recv", item, src) and ("prepare", item) for src == -1 (fetch / prefill)."""
    acts = []
    for item, src, dst, mode, _sec in moves:
        if src == rank:
            acts.append(("send", item, dst, mode))
        if dst == rank:
            acts.append(("recv", item, src) if src >= 0 else ("prepare", item))
    return acts


def execute_local(pools, wl, groups, moves, node_maps, stream=None):
    """Realise `moves` between pools of this process (pools[w] = worker w, same GPU and KV
    geometry).  node_maps[w] maps workload node ident -> node id in pools[w] (updated in
    place).  A group's nodes are cloned parents first (groups list them root first, DFS);
    a MOVE releases the source subtree afterwards (leaves first).  Moves with src == -1
    (no worker holds the KV) are skipped: the caller prepares those groups."""
    parent_of = {nd.ident: nd.parent for nd in wl.nodes}
    for item, src, dst, mode, _sec in moves:
        if src < 0:
            continue
        g = groups[item]
        for n in g.nodes:
            p = parent_of[n]
            new = pools[src].clone_prefix(node_maps[src][n], pools[dst],
                                          node_maps[dst][p] if p >= 0 else -1, stream)
            node_maps[dst][n] = new
        if mode == 0:
            for n in reversed(g.nodes):
                pools[src].release_prefix(node_maps[src].pop(n))
    return node_maps
