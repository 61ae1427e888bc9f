"""Multi-GPU partitioning of the decode batch (host logic only).

The attention of one (request, q-head) row depends only on that row's keys: the prefix
nodes on its path and its private suffix ("exact answers": sharing changes
where the work runs, not what it computes).  So the path shards with NO exchange step and
the only cross-GPU traffic is KV-block migration (NCCL send/recv).  Two
partitionings, as the paper's query sharding with operator replication (PAPER.md:236,
data-parallel baseline :601):

* request groups -- a prefix tree's root with every node and request under it stays on one
  rank (its K1 tiles need all of the node's requests); groups are placed by LPT over a cost
  model (prefix FLOPs / tensor peak + suffix bytes / HBM peak, the two rooflines of K1 and
  K2), deterministic tie-break by group index;
* kv heads -- rank p holds kv heads [p*H/P, (p+1)*H/P) of every block and serves their
  g*H/P q-heads; every rank runs the same plan on its head slice.

`max_over_ranks` is the timing reduction bench.py uses (device time, max over ranks).
"""
from __future__ import annotations

from dataclasses import dataclass

# roofline denominators for the placement cost (relative costs only; measured peaks are
# used when bench.py passes them in)
DEFAULT_TC_FLOPS = 1.675e15
DEFAULT_HBM_BPS = 6.5e12


@dataclass(frozen=True)
class Group:
    root: int            # root node ident (-1: the requests without a shared prefix)
    nodes: tuple         # node idents of the subtree (root first)
    requests: tuple      # request indices under the subtree
    cost: float          # seconds (per layer): prefix FLOPs / TC + suffix bytes / HBM


def subtree_groups(wl, tc_flops: float = DEFAULT_TC_FLOPS, hbm_bps: float = DEFAULT_HBM_BPS,
                   min_rows: int = 64) -> list:
    """One group per root node of the workload's prefix tree (+ one for prefix-less
    requests), with its per-layer cost.  A node whose requests give fewer than `min_rows`
    K1 rows is costed as folded into K2 (its KV bytes re-read per request), like the
    planner does."""
    children = {}
    for nd in wl.nodes:
        children.setdefault(nd.parent, []).append(nd.ident)
    ntok = {nd.ident: nd.ntok for nd in wl.nodes}
    under = {}   # node -> requests whose path contains it
    for r in wl.requests:
        for n in wl.path(r.ident):
            under.setdefault(n, []).append(r.ident)
    kv_tok = wl.hkv * wl.d * 2 * 2   # K+V bytes per token per layer
    groups = []
    for root in sorted(children.get(-1, [])):
        nodes, stack = [], [root]
        while stack:
            n = stack.pop()
            nodes.append(n)
            stack.extend(sorted(children.get(n, []), reverse=True))
        reqs = sorted(set(under.get(root, [])))
        flops, nbytes = 0.0, 0.0
        for n in nodes:
            rows = len(under.get(n, [])) * wl.g
            if rows >= min_rows:
                flops += 4.0 * rows * ntok[n] * wl.d * wl.hkv
                nbytes += ntok[n] * kv_tok
            else:
                nbytes += len(under.get(n, [])) * ntok[n] * kv_tok
        nbytes += sum(wl.requests[r].suffix + 1 for r in reqs) * kv_tok
        groups.append(Group(root, tuple(nodes), tuple(reqs), flops / tc_flops + nbytes / hbm_bps))
    loose = tuple(r.ident for r in wl.requests if r.leaf < 0)
    if loose:
        nbytes = sum(wl.requests[r].suffix + 1 for r in loose) * kv_tok
        groups.append(Group(-1, (), loose, nbytes / hbm_bps))
    return groups


def place_groups(costs, world: int) -> list:
    """LPT: groups in decreasing cost (ties: lower index first) to the least-loaded rank
    (ties: lower rank).  Returns the rank of every group."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0.0] * world
    rank_of = [0] * len(costs)
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        rank_of[i] = r
        load[r] += costs[i]
    return rank_of


def rank_requests(wl, world: int, rank: int, **kw) -> list:
    """Request indices this rank serves under request-group sharding."""
    groups = subtree_groups(wl, **kw)
    where = place_groups([g.cost for g in groups], world)
    return sorted(r for g, w in zip(groups, where) if w == rank for r in g.requests)


def head_range(hkv: int, world: int, rank: int) -> tuple:
    """kv heads [lo, hi) of `rank` under kv-head sharding (hkv divisible by world)."""
    if world < 1 or hkv % world:
        raise ValueError(f"{hkv} kv heads do not split over {world} ranks")
    per = hkv // world
    return rank * per, (rank + 1) * per


def max_over_ranks(values, dist=None, device=None) -> list:
    """Element-wise max of a list of floats over the process group (identity when
    single-process).  bench.py reduces its device times with it."""
    if dist is None or not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return list(values)
    import torch
    if dist.get_backend() == "gloo":
        device = "cpu"
    t = torch.tensor(list(values), dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def subset_workload(wl, requests, seed=None):
    """The sub-batch of `requests` (renumbered 0..n-1 in the given order) with the prefix
    nodes on their paths: the workload one rank serves under request-group sharding.
    Values are regenerated from (seed, node/request ident), so only the structure carries
    over (a benchmark shard, not a slice of the parent's tensors)."""
    from synth.workloads import RequestSpec, Workload
    keep = set()
    for r in requests:
        keep.update(wl.path(r))
    nodes = [nd for nd in wl.nodes if nd.ident in keep]
    reqs = [RequestSpec(i, wl.requests[r].leaf, wl.requests[r].suffix) for i, r in enumerate(requests)]
    return Workload(wl.name, wl.layers, wl.hq, wl.hkv, wl.d, nodes, reqs,
                    wl.seed if seed is None else seed, alpha_q=wl.alpha_q)


def head_shard_workload(wl, world: int, rank: int):
    """The same batch with this rank's kv heads (and their q-heads) only."""
    from synth.workloads import Workload
    lo, hi = head_range(wl.hkv, world, rank)
    return Workload(wl.name, wl.layers, wl.g * (hi - lo), hi - lo, wl.d, list(wl.nodes),
                    list(wl.requests), wl.seed, alpha_q=wl.alpha_q)
