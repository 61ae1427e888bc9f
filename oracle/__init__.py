"""fp64 CPU oracle for shared-prefix decode attention -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` leg
may import this package.  The product package (paper_2509_02121_b200) never imports it and
the two share no code; the only common import is the seeded input generator `synth`, which
holds no attention arithmetic.

Functions and the passages they follow:
  attend(...)          -- unshared softmax attention, fp64 C (attend.c).
                          (§2.2 "Exact answers": optimised == naive execution), :343
                          (§3.3 prefix caching = reuse of precomputed state); SURVEY.md
                          §8(c) steps 1-6.
  request_context(...) -- step 2 of §8(c): the key/value list of a request is the
                          concatenation of its prefix path root -> leaf (the shared
                          prefixes of the consolidated DAG) followed by
                          its private suffix and the tokens appended by decode steps
                          (decode reuses cached K/V, §2.1).
  decode_reference(...)-- attend() over request_context() for a set of requests.
  lse_merge(...)       -- the log-sum-exp combination of partial softmax states.  It is
                          the algebra behind reusing a cached prefix without changing the
                          answer; pinned in tests against the unshared
                          definition (shared == unshared), associativity, commutativity
                          and the -inf identity.

Every function is pinned in tests/test_oracle.py against closed forms, invariants, a
hand-derived golden example (tests/golden/) and torch's float64 SDPA; see DESIGN.md
"Oracle pins".  Nothing here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "attend.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile attend.c with gcc (no -ffast-math).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c11",
                               "-Wall", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_attend.restype = ctypes.c_int
        lib.oracle_attend.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_int]
        _lib = lib
    return _lib


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def attend(q_bits: np.ndarray, k_bits: np.ndarray, v_bits: np.ndarray, scale: float,
           nthreads: int | None = None):
    """q [hq][d], k/v [T][hkv][d] as uint16 bf16 bit patterns -> (out [hq][d], lse [hq])."""
    lib = _load()
    q = np.ascontiguousarray(q_bits, dtype=np.uint16)
    k = np.ascontiguousarray(k_bits, dtype=np.uint16)
    v = np.ascontiguousarray(v_bits, dtype=np.uint16)
    hq, d = q.shape
    T, hkv, d2 = k.shape
    assert d2 == d and v.shape == k.shape
    out = np.empty((hq, d), dtype=np.float64)
    lse = np.empty((hq,), dtype=np.float64)
    rc = lib.oracle_attend(T, hq, hkv, d, q.ctypes.data, k.ctypes.data, v.ctypes.data,
                           float(scale), out.ctypes.data, lse.ctypes.data,
                           int(nthreads or default_threads()))
    if rc != 0:
        raise ValueError("oracle_attend rejected its arguments")
    return out, lse


def _bits(t) -> np.ndarray:
    import torch
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def request_context(wl, r: int, layer: int, steps: int = 1, cache: dict | None = None):
    """(k_bits, v_bits) [T][Hkv][d] for request r at `layer` after `steps` decode steps:
    prefix path root -> leaf, then the initial suffix, then the appended tokens.
    `cache` (optional) memoises the generated prefix-node tensors across requests."""
    ks, vs = [], []
    for n in wl.path(r):
        key = (n, layer)
        if cache is not None and key in cache:
            k, v = cache[key]
        else:
            k, v = wl.node_kv(n, "cpu", layer)
            k, v = _bits(k), _bits(v)
            if cache is not None:
                cache[key] = (k, v)
        ks.append(k)
        vs.append(v)
    k, v = wl.suffix_kv("cpu", layer, request=r)
    ks.append(_bits(k))
    vs.append(_bits(v))
    for s in range(steps):
        k, v = wl.new_kv(s, "cpu", layer, request=r)
        ks.append(_bits(k)[None])
        vs.append(_bits(v)[None])
    return np.concatenate(ks, axis=0), np.concatenate(vs, axis=0)


def decode_reference(wl, layer: int, steps: int = 1, requests=None, scale=None,
                     nthreads: int | None = None):
    """fp64 (out [n][Hq][d], lse [n][Hq]) of decode step `steps-1` for `requests`."""
    if requests is None:
        requests = range(wl.nreq)
    requests = list(requests)
    if scale is None:
        scale = 1.0 / np.sqrt(wl.d)
    out = np.empty((len(requests), wl.hq, wl.d), dtype=np.float64)
    lse = np.empty((len(requests), wl.hq), dtype=np.float64)
    cache = {}
    for i, r in enumerate(requests):
        k, v = request_context(wl, r, layer, steps, cache)
        q = _bits(wl.q(steps - 1, "cpu", layer, request=r))
        out[i], lse[i] = attend(q, k, v, scale, nthreads)
    return out, lse


def lse_merge(outs, lses):
    """Combine partial softmax states (o_i normalised, lse_i natural log) of disjoint key
    sets into the state of their union:
        m = max_i lse_i;  w_i = exp(lse_i - m);  o = sum_i w_i o_i / sum_i w_i;
        lse = m + ln sum_i w_i.
    A partial with lse = -inf (empty key set) is the identity.  Shapes: outs [n][..., d],
    lses [n][...]."""
    outs = np.asarray(outs, dtype=np.float64)
    lses = np.asarray(lses, dtype=np.float64)
    m = np.max(lses, axis=0)
    m_safe = np.where(np.isfinite(m), m, 0.0)
    w = np.where(np.isfinite(lses), np.exp(lses - m_safe), 0.0)
    tot = np.sum(w, axis=0)
    with np.errstate(invalid="ignore", divide="ignore"):
        o = np.sum(w[..., None] * outs, axis=0) / tot[..., None]
        lse = m_safe + np.log(tot)
    empty = ~np.isfinite(m)
    o = np.where(empty[..., None], 0.0, o)
    lse = np.where(empty, -np.inf, lse)
    return o, lse
