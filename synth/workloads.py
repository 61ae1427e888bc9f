"""Synthetic workloads shaped like the paper's benchmarks (BASELINE.json `configs`).

A workload is a prefix tree of shared KV segments plus a batch of decode requests:
  * nodes  — shared prefix segments (workflow template -> role -> ...); the tree induced by
             the consolidated query-plan DAG (PAPER.md:54 §1, :273 §3.1 example; template
             fan-out :135 §2.2; fan-out/fan-in primitives :296-302 §3.2),
  * requests — each hangs under one leaf node (or none) and owns a private suffix.
Values come from `synth.gen` (counter-based, identical on CPU and GPU).  Nothing here does
attention arithmetic.

Decode-step convention (reading R4): a step appends ONE new token per request
(K/V from `new_kv(step)`) and then attends with `q(step)`; the attended context of request
r after step s is  path(r) nodes ++ initial suffix ++ new tokens of steps 0..s.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .gen import TensorKey, bf16_tensor


@dataclass(frozen=True)
class NodeSpec:
    ident: int
    parent: int  # -1 for a root
    ntok: int


@dataclass(frozen=True)
class RequestSpec:
    ident: int
    leaf: int     # -1: no shared prefix
    suffix: int   # private tokens present before the first decode step


@dataclass
class Workload:
    name: str
    layers: int
    hq: int
    hkv: int
    d: int
    nodes: list
    requests: list
    seed: int = 0
    alpha_q: float = 1.0
    # attention-sink variant (SURVEY.md §8(d) "sink (+8 on token 0 of the root)"): token 0
    # of every root node gets the key K0 * e_0 and every query gets +SINK_QB on dim 0, so its
    # scaled score is sink * (1 + z * alpha / SINK_QB) with z ~ N(0,1): +sink on average.
    sink: float = 0.0
    # value distribution of every tensor (synth.gen: "grid" = round-1 multiples of 1/32,
    # "normal" = bf16(N(0,1)) with a full mantissa)
    dist: str = "grid"
    # outlier channels: K (nodes, suffixes, new tokens) dims in `k_outlier_dims` x 2^k_outlier_log2
    k_outlier_dims: tuple = ()
    k_outlier_log2: int = 6
    # V magnitude per prefix node: node ident -> p, its V x 2^p (exact); requests whose leaf
    # is that node get the same factor on their suffix and appended V (the whole context of
    # such a request is scaled, so its exact output scales by 2^p: o(aV) = a o(V))
    v_scale_log2: dict = field(default_factory=dict)
    # within a node: node ident -> (tok0, p): its tokens [tok0, ntok) get an extra V x 2^p
    v_token_scale_log2: dict = field(default_factory=dict)
    notes: dict = field(default_factory=dict)

    # ---- structure -------------------------------------------------------------------
    @property
    def g(self) -> int:
        return self.hq // self.hkv

    @property
    def nreq(self) -> int:
        return len(self.requests)

    def node(self, ident: int) -> NodeSpec:
        return self._nodes_by_id[ident]

    def __post_init__(self):
        self._nodes_by_id = {n.ident: n for n in self.nodes}
        assert self.hq % self.hkv == 0
        offs = np.zeros(len(self.requests) + 1, dtype=np.int64)
        for i, r in enumerate(self.requests):
            offs[i + 1] = offs[i] + r.suffix
        self.suffix_offsets = offs

    def path(self, r: int) -> list:
        """Node ids root -> leaf for request index r."""
        out = []
        n = self.requests[r].leaf
        while n != -1:
            out.append(n)
            n = self._nodes_by_id[n].parent
        return out[::-1]

    def context_len(self, r: int, steps: int = 1) -> int:
        return sum(self.node(n).ntok for n in self.path(r)) + self.requests[r].suffix + steps

    # ---- tensors (layout [layer][token][head][d], bf16) -------------------------------
    def _key(self, kind: str, ident: int) -> TensorKey:
        return TensorKey(self.seed, kind, ident)

    SINK_QB = 4.0  # query bias on dim 0 of the sink variant

    # ---- value shaping (exact: powers of two) -----------------------------------------
    def _k_out(self, k):
        if self.k_outlier_dims:
            k = k.clone()
            idx = list(self.k_outlier_dims)
            k[..., idx] = (k[..., idx].float() * 2.0 ** self.k_outlier_log2).to(torch.bfloat16)
        return k

    def _v_scale(self, v, leaf_of_rows=None, node=None):
        """Scale V by 2^p: of node `node`, or per row (dim -3) by the scale of each row's leaf."""
        if not self.v_scale_log2:
            return v
        if node is not None:
            p = self.v_scale_log2.get(node, 0)
            return v if p == 0 else (v.float() * 2.0 ** p).to(torch.bfloat16)
        f = torch.tensor([2.0 ** self.v_scale_log2.get(lf, 0) for lf in leaf_of_rows],
                         dtype=torch.float32, device=v.device)
        return (v.float() * f[:, None, None]).to(torch.bfloat16)

    def _row_leaves(self, request=None):
        """Leaf of every initial-suffix token row (or of request `request`'s rows)."""
        if request is not None:
            return [self.requests[request].leaf] * self.requests[request].suffix
        return [r.leaf for r in self.requests for _ in range(r.suffix)]

    def node_kv(self, n: int, device="cpu", layer=None):
        nt = self.node(n).ntok
        k, v = self._pair("node_k", "node_v", n, nt, self.hkv, device, layer)
        k, v = self._k_out(k), self._v_scale(v, node=n)
        if n in self.v_token_scale_log2:
            t0, p = self.v_token_scale_log2[n]
            v = v.clone()
            if layer is None:
                v[:, t0:] = (v[:, t0:].float() * 2.0 ** p).to(torch.bfloat16)
            else:
                v[t0:] = (v[t0:].float() * 2.0 ** p).to(torch.bfloat16)
        if self.sink > 0 and self.node(n).parent < 0:
            # K0 = sink * sqrt(d) / SINK_QB on dim 0, zero elsewhere (exact in bf16 after rounding)
            k0 = torch.zeros(self.hkv, self.d, dtype=torch.float32)
            k0[:, 0] = self.sink * (self.d ** 0.5) / self.SINK_QB
            k0 = k0.to(torch.bfloat16).to(k.device)
            if layer is None:
                k[:, 0] = k0
            else:
                k[0] = k0
        return k, v

    def suffix_kv(self, device="cpu", layer=None, request=None):
        """Initial suffixes of all requests: [L][sum S][Hkv][d], or one request's slice."""
        tot = int(self.suffix_offsets[-1])
        row = self.hkv * self.d
        if request is None:
            k, v = self._pair("suf_k", "suf_v", 0, tot, self.hkv, device, layer)
            if self.v_scale_log2:
                lv = self._row_leaves()
                v = self._v_scale(v, lv) if layer is not None else \
                    torch.stack([self._v_scale(v[i], lv) for i in range(v.shape[0])])
            return self._k_out(k), v
        s0, s1 = int(self.suffix_offsets[request]), int(self.suffix_offsets[request + 1])
        assert layer is not None
        off = (layer * tot + s0) * row
        shape = (s1 - s0, self.hkv, self.d)
        k = bf16_tensor(self._key("suf_k", 0), shape, device, off, dist=self.dist)
        v = bf16_tensor(self._key("suf_v", 0), shape, device, off, dist=self.dist)
        return self._k_out(k), self._v_scale(v, self._row_leaves(request))

    def q(self, step: int, device="cpu", layer=None, request=None):
        """Decode queries of step `step`: [L][R][Hq][d] (or a slice)."""
        q = self._rows("q", step, self.hq, device, layer, request, self.alpha_q)
        if self.sink > 0:  # + SINK_QB on dim 0, rounded to bf16 (same on CPU and GPU)
            q[..., 0] = (q[..., 0].float() + self.SINK_QB).to(torch.bfloat16)
        return q

    def new_kv(self, step: int, device="cpu", layer=None, request=None):
        """K/V of the token appended at step `step`: [L][R][Hkv][d] (or a slice)."""
        k = self._k_out(self._rows("new_k", step, self.hkv, device, layer, request))
        v = self._rows("new_v", step, self.hkv, device, layer, request)
        if self.v_scale_log2:
            if request is not None:
                v = self._v_scale(v[None], [self.requests[request].leaf])[0]
            else:
                lv = [r.leaf for r in self.requests]
                v = self._v_scale(v, lv) if layer is not None else \
                    torch.stack([self._v_scale(v[i], lv) for i in range(v.shape[0])])
        return k, v

    def _pair(self, kk, kv, ident, ntok, heads, device, layer):
        row = heads * self.d
        if layer is None:
            shape, off = (self.layers, ntok, heads, self.d), 0
        else:
            shape, off = (ntok, heads, self.d), layer * ntok * row
        return (bf16_tensor(self._key(kk, ident), shape, device, off, dist=self.dist),
                bf16_tensor(self._key(kv, ident), shape, device, off, dist=self.dist))

    def _rows(self, kind, ident, heads, device, layer, request, alpha=1.0):
        R = self.nreq
        row = heads * self.d
        if layer is None:
            assert request is None
            return bf16_tensor(self._key(kind, ident), (self.layers, R, heads, self.d), device,
                               0, alpha, dist=self.dist)
        if request is None:
            return bf16_tensor(self._key(kind, ident), (R, heads, self.d), device,
                               layer * R * row, alpha, dist=self.dist)
        return bf16_tensor(self._key(kind, ident), (heads, self.d), device,
                           (layer * R + request) * row, alpha, dist=self.dist)


# ---------------------------------------------------------------------------------------
# Config builders.  C0..C4 follow BASELINE.json `configs`; the small
# parity variants keep the same structure at sizes the fp64 oracle finishes in seconds.
# ---------------------------------------------------------------------------------------

def _fanout(name, layers, hq, hkv, d, nreq, prefix, suffix, seed, **kw):
    nodes = [NodeSpec(0, -1, prefix)] if prefix > 0 else []
    leaf = 0 if prefix > 0 else -1
    reqs = [RequestSpec(i, leaf, suffix) for i in range(nreq)]
    return Workload(name, layers, hq, hkv, d, nodes, reqs, seed, **kw)


def toy(seed=0, **kw):
    """C0: 4 requests share a 64-token prefix, 16-token suffixes (15 + the decoded token),
    1 head, d=64."""
    return _fanout("toy", 1, 1, 1, 64, 4, 64, 15, seed, **kw)


def fanout(seed=1, layers=32, nreq=256, prefix=2048, suffix=255, hq=32, hkv=8, d=128, **kw):
    """C1: Llama-3-8B GQA; `nreq` requests fanned out from one template prefix.  The
    suffix is 255 initial tokens + the decoded token = 256 attended suffix tokens."""
    return _fanout("fanout", layers, hq, hkv, d, nreq, prefix, suffix, seed, **kw)


def tree(seed=2, layers=32, root=4096, roles=16, role_tok=1024, per_role=64, suffix=255,
         hq=32, hkv=8, d=128, **kw):
    """C2: system prompt -> role prefixes -> requests (consolidated agent DAG)."""
    nodes = [NodeSpec(0, -1, root)] + [NodeSpec(1 + i, 0, role_tok) for i in range(roles)]
    reqs = [RequestSpec(i, 1 + i // per_role, suffix) for i in range(roles * per_role)]
    return Workload("tree", layers, hq, hkv, d, nodes, reqs, seed, **kw)


def analytics(seed=3, layers=32, templates=8, ctx=8192, per_template=256, suffix=255,
              hq=32, hkv=8, d=128, **kw):
    """C3: batch analytics; `templates` independent shared contexts (8 per GPU of 64)."""
    nodes = [NodeSpec(i, -1, ctx) for i in range(templates)]
    reqs = [RequestSpec(i, i // per_template, suffix) for i in range(templates * per_template)]
    return Workload("analytics", layers, hq, hkv, d, nodes, reqs, seed, **kw)


def ragged(seed=4, layers=2, hq=8, hkv=2, d=128, **kw):
    """Parity stress: a depth-3 tree with partial blocks, requests without a prefix,
    ragged suffixes (incl. 0 initial tokens), and one node shared by a single request."""
    rng = np.random.Generator(np.random.PCG64(1000 + seed))
    nodes = [NodeSpec(0, -1, 301), NodeSpec(1, 0, 77), NodeSpec(2, 0, 160),
             NodeSpec(3, 1, 33), NodeSpec(4, -1, 5), NodeSpec(5, 2, 129)]
    leaves = [0, 1, 2, 3, 3, 3, 4, 5, -1, 2, 1, 5, 3, 0, -1, 2] * 3
    reqs = []
    for i, lf in enumerate(leaves):
        s = int(rng.integers(0, 300)) if i % 7 else 0
        reqs.append(RequestSpec(i, lf, s))
    return Workload("ragged", layers, hq, hkv, d, nodes, reqs, seed, **kw)


def ragged_suffix(seed=5, layers=2, nreq=96, prefix=1024, lo=128, hi=1024, hq=32, hkv=8,
                  d=128, **kw):
    """C1 variant with S_r ~ U[lo, hi] (the output-length range of PAPER.md:685 §4.5)."""
    rng = np.random.Generator(np.random.PCG64(2000 + seed))
    nodes = [NodeSpec(0, -1, prefix)]
    reqs = [RequestSpec(i, 0, int(rng.integers(lo, hi + 1)) - 1) for i in range(nreq)]
    return Workload("ragged_suffix", layers, hq, hkv, d, nodes, reqs, seed, **kw)


def scaled(seed=6, layers=2, hq=8, hkv=2, d=128, dist="normal", **kw):
    """V-range stress (K1 converts V to fp16 for the P.V MMA): three roots -- unit-scale V
    whose tokens 600.. are x 2^20 (the fp16 scale must grow inside a tile), V x 2^17 (|V| up to ~8e5, beyond fp16's 65504) and V x 2^-22 (|V| <= ~1.4e-6, below
    fp16's normal range) -- plus a unit-scale child under the huge root, requests on every
    node with ragged suffixes scaled like their leaf; full-mantissa normal values."""
    nodes = [NodeSpec(0, -1, 1000), NodeSpec(1, -1, 777), NodeSpec(2, -1, 640),
             NodeSpec(3, 1, 300)]
    reqs = [RequestSpec(i, i % 4, 20 + 37 * (i % 5)) for i in range(64)]
    kw.setdefault("v_scale_log2", {1: 17, 2: -22})
    kw.setdefault("v_token_scale_log2", {0: (600, 20)})  # V grows x 2^20 mid-node
    return Workload("scaled", layers, hq, hkv, d, nodes, reqs, seed, dist=dist, **kw)


def tree_root(seed=2, layers=32, **kw):
    """C2's root node class alone: 1024 requests under one 4096-token prefix (K1 rows 4096 per
    kv head, arithmetic intensity 4096) -- the C2-root K1 gate of SURVEY.md §8(d)."""
    return _fanout("tree_root", layers, 32, 8, 128, 1024, 4096, 255, seed, **kw)


def tree_roles(seed=2, layers=32, **kw):
    """C2's role node class alone: 16 prefixes of 1024 tokens with 64 requests each (K1 rows
    256 per kv head, arithmetic intensity 256 ~ the ridge)."""
    nodes = [NodeSpec(i, -1, 1024) for i in range(16)]
    reqs = [RequestSpec(i, i // 64, 255) for i in range(1024)]
    return Workload("tree_roles", layers, 32, 8, 128, nodes, reqs, seed, **kw)


CONFIGS = {
    "tree_root": tree_root,
    "tree_roles": tree_roles,
    "scaled": scaled,
    "toy": toy,
    "fanout": fanout,
    "tree": tree,
    "analytics": analytics,
    "ragged": ragged,
    "ragged_suffix": ragged_suffix,
}


def make_config(name: str, **kw) -> Workload:
    return CONFIGS[name](**kw)
