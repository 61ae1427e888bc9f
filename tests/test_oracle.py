"""Pins of the fp64 oracle against things other than itself (closed forms, invariants,
hand-derived golden values, torch's float64 SDPA, 50-digit brute force).

Each pin is chosen so that a plausible mistake in oracle/attend.c or oracle/__init__.py
fails at least one test:
  * dropped scale / wrong scale placement   -> golden, single-token, key-shift, SDPA
  * wrong GQA mapping (h % hkv vs h // g)   -> golden GQA case, SDPA with 2+ kv heads
  * transposed operands / wrong strides     -> SDPA on random tensors, golden
  * max not subtracted consistently / lse   -> golden lse, duplicate-token ln 2, q=0 ln T
  * missing normalisation by Z              -> q=0 mean(V), affine-in-V
  * dropped prefix node or suffix in gather -> shared==unshared, context-length checks
  * wrong merge weights / -inf handling     -> golden merge, associativity, identity
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from synth import make_config
from synth.gen import bf16_bits, bf16_tensor, TensorKey

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hand_examples.json")


def to_bits(x) -> np.ndarray:
    """float array of bf16-representable values -> bf16 bit patterns (asserts exactness)."""
    t = torch.as_tensor(np.asarray(x, dtype=np.float32))
    b = t.to(torch.bfloat16)
    assert torch.equal(b.to(torch.float32), t), "value not bf16-representable"
    return bf16_bits(b)


def f64(bits):
    return (np.asarray(bits, dtype=np.uint32) << 16).view(np.float32).astype(np.float64)


def rand_bits(shape, seed, alpha=1.0):
    return bf16_bits(bf16_tensor(TensorKey(seed, "q", 99), shape, alpha=alpha))


# ---------------------------------------------------------------- golden (hand-derived)
def test_golden_attend():
    doc = json.load(open(GOLDEN))
    for case in doc["attend"]:
        out, lse = oracle.attend(to_bits(case["q"]), to_bits(case["k"]), to_bits(case["v"]),
                                 case["scale"], nthreads=2)
        np.testing.assert_allclose(out, np.array(case["out"]), rtol=0, atol=1e-14,
                                   err_msg=case["what"])
        np.testing.assert_allclose(lse, np.array(case["lse"]), rtol=0, atol=1e-14,
                                   err_msg=case["what"])


def test_golden_merge():
    doc = json.load(open(GOLDEN))
    for case in doc["merge"]:
        lses = [float(x) for x in case["lses"]]
        o, lse = oracle.lse_merge(np.array(case["outs"]), np.array(lses))
        np.testing.assert_allclose(o, case["out"], atol=1e-14, err_msg=case["what"])
        assert abs(lse - case["lse"]) < 1e-14, case["what"]


# ---------------------------------------------------------------- closed forms
def test_single_token_is_value():
    q, k, v = rand_bits((4, 16), 1), rand_bits((1, 2, 16), 2), rand_bits((1, 2, 16), 3)
    out, lse = oracle.attend(q, k, v, 0.25)
    qf, kf, vf = f64(q), f64(k), f64(v)
    for h in range(4):
        j = h // 2
        assert np.array_equal(out[h], vf[0, j])
        assert abs(lse[h] - 0.25 * float(qf[h] @ kf[0, j])) < 1e-12


def test_zero_query_is_mean_value():
    T = 37
    q = np.zeros((2, 8), dtype=np.uint16)  # +0.0 in bf16
    k, v = rand_bits((T, 1, 8), 4), rand_bits((T, 1, 8), 5)
    out, lse = oracle.attend(q, k, v, 0.7)
    np.testing.assert_allclose(out[0], f64(v)[:, 0].mean(axis=0), atol=1e-14)
    np.testing.assert_allclose(lse, math.log(T), atol=1e-14)


def test_equal_keys_is_mean_value():
    T = 19
    q = rand_bits((1, 8), 6)
    k = np.repeat(rand_bits((1, 1, 8), 7), T, axis=0)
    v = rand_bits((T, 1, 8), 8)
    out, lse = oracle.attend(q, k, v, 0.3)
    s = 0.3 * float(f64(q)[0] @ f64(k)[0, 0])
    np.testing.assert_allclose(out[0], f64(v)[:, 0].mean(axis=0), atol=1e-13)
    assert abs(lse[0] - (s + math.log(T))) < 1e-12


def test_duplicated_tokens_add_ln2():
    q, k, v = rand_bits((4, 32), 9), rand_bits((50, 2, 32), 10), rand_bits((50, 2, 32), 11)
    o1, l1 = oracle.attend(q, k, v, 0.2)
    o2, l2 = oracle.attend(q, np.concatenate([k, k]), np.concatenate([v, v]), 0.2)
    np.testing.assert_allclose(o2, o1, atol=1e-13)
    np.testing.assert_allclose(l2, l1 + math.log(2.0), atol=1e-12)


def test_dominant_score_selects_value():
    # token 5 has a score gap >= 800 over every other token: exp(-800) underflows to 0.
    T, d = 12, 8
    q = to_bits(np.ones((1, d)))
    kk = np.zeros((T, 1, d))
    kk[5] = 128.0
    k, v = to_bits(kk), rand_bits((T, 1, d), 12)
    out, _ = oracle.attend(q, k, v, 1.0)
    assert np.array_equal(out[0], f64(v)[5, 0])


def test_affine_in_values():
    q, k, v = rand_bits((2, 16), 13), rand_bits((40, 1, 16), 14), rand_bits((40, 1, 16), 15)
    o1, l1 = oracle.attend(q, k, v, 0.25)
    v2 = to_bits(2.0 * f64(v) + 0.5)  # exact in bf16 for these small integers/32
    o2, l2 = oracle.attend(q, k, v2, 0.25)
    np.testing.assert_allclose(o2, 2.0 * o1 + 0.5, atol=1e-12)
    np.testing.assert_allclose(l2, l1, atol=0)


def test_key_shift_moves_lse_only():
    d = 16
    q, k, v = rand_bits((2, d), 16), rand_bits((30, 1, d), 17), rand_bits((30, 1, d), 18)
    c = np.zeros(d)
    c[3] = 1.0
    c[7] = -2.0
    k2 = to_bits(f64(k) + c)
    o1, l1 = oracle.attend(q, k, v, 0.5)
    o2, l2 = oracle.attend(q, k2, v, 0.5)
    np.testing.assert_allclose(o2, o1, atol=1e-12)
    np.testing.assert_allclose(l2, l1 + 0.5 * (f64(q) @ c), atol=1e-12)


def test_empty_context_is_merge_identity():
    out, lse = oracle.attend(rand_bits((2, 8), 19), np.zeros((0, 1, 8), np.uint16),
                             np.zeros((0, 1, 8), np.uint16), 1.0)
    assert np.all(out == 0) and np.all(np.isneginf(lse))


# ---------------------------------------------------------------- library routine
def sdpa_reference(q, k, v, scale):
    """torch float64 SDPA with HF repeat_kv (q-head h -> kv head h // g)."""
    qf = torch.from_numpy(f64(q))            # [hq, d]
    kf = torch.from_numpy(f64(k))            # [T, hkv, d]
    vf = torch.from_numpy(f64(v))
    hq, hkv = qf.shape[0], kf.shape[1]
    kr = kf.permute(1, 0, 2).repeat_interleave(hq // hkv, dim=0)  # [hq, T, d]
    vr = vf.permute(1, 0, 2).repeat_interleave(hq // hkv, dim=0)
    o = torch.nn.functional.scaled_dot_product_attention(qf[:, None, :], kr, vr, scale=scale)
    lse = torch.logsumexp(scale * torch.einsum("hd,htd->ht", qf, kr), dim=1)
    return o[:, 0, :].numpy(), lse.numpy()


@pytest.mark.parametrize("hq,hkv,d,T,alpha", [(32, 8, 128, 333, 1.0), (8, 2, 64, 70, 2.0),
                                               (4, 4, 16, 5, 4.0), (6, 3, 32, 1000, 1.0)])
def test_matches_torch_sdpa(hq, hkv, d, T, alpha):
    q = rand_bits((hq, d), 20 + T, alpha)
    k, v = rand_bits((T, hkv, d), 21 + T), rand_bits((T, hkv, d), 22 + T)
    scale = 1.0 / math.sqrt(d)
    out, lse = oracle.attend(q, k, v, scale)
    ro, rl = sdpa_reference(q, k, v, scale)
    np.testing.assert_allclose(out, ro, atol=1e-12)
    np.testing.assert_allclose(lse, rl, atol=1e-12)


# ---------------------------------------------------------------- 50-digit brute force
def test_mpmath_brute_force():
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 50
    for trial in range(6):
        hq, hkv, d, T = 4, 2, 4, 3 + 2 * trial
        q, k, v = rand_bits((hq, d), 30 + trial, 2.0), rand_bits((T, hkv, d), 40 + trial), \
            rand_bits((T, hkv, d), 50 + trial)
        scale = 0.5
        out, lse = oracle.attend(q, k, v, scale)
        qf, kf, vf = f64(q), f64(k), f64(v)
        for h in range(hq):
            j = h * hkv // hq
            s = [mpmath.mpf(scale) * mpmath.fsum(mpmath.mpf(qf[h, i]) * mpmath.mpf(kf[t, j, i])
                                                 for i in range(d)) for t in range(T)]
            w = [mpmath.e ** x for x in s]
            Z = mpmath.fsum(w)
            for i in range(d):
                ref = mpmath.fsum(w[t] * mpmath.mpf(vf[t, j, i]) for t in range(T)) / Z
                assert abs(out[h, i] - float(ref)) < 1e-13
            assert abs(lse[h] - float(mpmath.log(Z))) < 1e-13


# ---------------------------------------------------------------- invariants
def test_token_permutation_invariance():
    q, k, v = rand_bits((8, 32), 60), rand_bits((90, 2, 32), 61), rand_bits((90, 2, 32), 62)
    perm = np.random.Generator(np.random.PCG64(7)).permutation(90)
    o1, l1 = oracle.attend(q, k, v, 0.2)
    o2, l2 = oracle.attend(q, k[perm], v[perm], 0.2)
    np.testing.assert_allclose(o2, o1, atol=1e-13)
    np.testing.assert_allclose(l2, l1, atol=1e-13)


def test_merge_algebra():
    rng = np.random.Generator(np.random.PCG64(3))
    parts = [(rng.standard_normal((3, 5)), rng.standard_normal(3) * 4) for _ in range(4)]
    parts.append((np.zeros((3, 5)), np.full(3, -np.inf)))
    o_all, l_all = oracle.lse_merge([p[0] for p in parts], [p[1] for p in parts])
    # commutativity
    for perm in itertools.permutations(range(5)):
        o, l = oracle.lse_merge([parts[i][0] for i in perm], [parts[i][1] for i in perm])
        np.testing.assert_allclose(o, o_all, atol=1e-13)
        np.testing.assert_allclose(l, l_all, atol=1e-13)
    # associativity: ((0,1),(2,3,4)) == all
    a = oracle.lse_merge([parts[0][0], parts[1][0]], [parts[0][1], parts[1][1]])
    b = oracle.lse_merge([p[0] for p in parts[2:]], [p[1] for p in parts[2:]])
    o, l = oracle.lse_merge([a[0], b[0]], [a[1], b[1]])
    np.testing.assert_allclose(o, o_all, atol=1e-13)
    np.testing.assert_allclose(l, l_all, atol=1e-13)
    # identity
    o, l = oracle.lse_merge([parts[0][0], parts[4][0]], [parts[0][1], parts[4][1]])
    np.testing.assert_allclose(o, parts[0][0], atol=0)
    np.testing.assert_allclose(l, parts[0][1], atol=0)


def test_split_point_invariance():
    """Attention over a token range == LSE merge of its two halves, for every split."""
    q, k, v = rand_bits((4, 16), 70), rand_bits((40, 2, 16), 71), rand_bits((40, 2, 16), 72)
    o_all, l_all = oracle.attend(q, k, v, 0.25)
    for c in range(0, 41, 3):
        a = oracle.attend(q, k[:c], v[:c], 0.25)
        b = oracle.attend(q, k[c:], v[c:], 0.25)
        o, l = oracle.lse_merge([a[0], b[0]], [a[1], b[1]])
        np.testing.assert_allclose(o, o_all, atol=1e-13)
        np.testing.assert_allclose(l, l_all, atol=1e-13)


def test_prefix_shared_equals_unshared():
    """The paper's exactness requirement: cascade evaluation (one partial per
    prefix node on the path + one for the private suffix, LSE-merged) == unshared oracle."""
    wl = make_config("ragged", layers=1)
    scale = 1.0 / math.sqrt(wl.d)
    out, lse = oracle.decode_reference(wl, 0, steps=1, scale=scale)
    for r in range(wl.nreq):
        q = bf16_bits(wl.q(0, "cpu", 0, request=r))
        parts_o, parts_l = [], []
        for n in wl.path(r):
            k, v = wl.node_kv(n, "cpu", 0)
            o, l = oracle.attend(q, bf16_bits(k), bf16_bits(v), scale)
            parts_o.append(o)
            parts_l.append(l)
        ks, vs = wl.suffix_kv("cpu", 0, request=r)
        nk, nv = wl.new_kv(0, "cpu", 0, request=r)
        k = np.concatenate([bf16_bits(ks), bf16_bits(nk)[None]])
        v = np.concatenate([bf16_bits(vs), bf16_bits(nv)[None]])
        o, l = oracle.attend(q, k, v, scale)
        parts_o.append(o)
        parts_l.append(l)
        mo, ml = oracle.lse_merge(parts_o, parts_l)
        np.testing.assert_allclose(mo, out[r], atol=1e-12)
        np.testing.assert_allclose(ml, lse[r], atol=1e-12)


def test_request_permutation_permutes_rows():
    wl = make_config("ragged", layers=1)
    perm = list(np.random.Generator(np.random.PCG64(11)).permutation(wl.nreq)[:12])
    out, lse = oracle.decode_reference(wl, 0, requests=range(wl.nreq))
    out_p, lse_p = oracle.decode_reference(wl, 0, requests=perm)
    assert np.array_equal(out_p, out[perm]) and np.array_equal(lse_p, lse[perm])


def test_context_is_path_then_suffix_then_new_tokens():
    wl = make_config("ragged", layers=2)
    for r in range(wl.nreq):
        k, v = oracle.request_context(wl, r, 1, steps=2)
        assert k.shape[0] == wl.context_len(r, steps=2)
        off = 0
        for n in wl.path(r):
            nk, _ = wl.node_kv(n, "cpu", 1)
            assert np.array_equal(k[off:off + nk.shape[0]], bf16_bits(nk))
            off += nk.shape[0]
        sk, _ = wl.suffix_kv("cpu", 1, request=r)
        assert np.array_equal(k[off:off + sk.shape[0]], bf16_bits(sk))


def test_generator_is_device_independent_and_seeded():
    key = TensorKey(5, "node_k", 3)
    a = bf16_tensor(key, (1000,))
    b = bf16_tensor(key, (400,), offset=600)
    assert torch.equal(a[600:], b)
    c = bf16_tensor(TensorKey(6, "node_k", 3), (1000,))
    assert not torch.equal(a, c)
    x = a.float()
    assert abs(float(x.mean())) < 0.15 and 0.9 < float(x.std()) < 1.4
    assert torch.equal((x * 32).round(), x * 32)  # multiples of 1/32: bf16-exact


def test_sink_variant_inputs():
    """The sink workload (inputs only): token 0 of a root carries K0 e_0 and every query has
    +4 on dim 0, so token 0's scaled score averages +sink; other tokens stay centred; the
    node tensors read per layer equal the all-layer read."""
    wl = make_config("fanout", layers=2, nreq=16, prefix=40, suffix=3, sink=8.0)
    k, _ = wl.node_kv(0, "cpu")
    for layer in range(2):
        kl, _ = wl.node_kv(0, "cpu", layer)
        assert torch.equal(kl, k[layer])
        q = wl.q(0, "cpu", layer).double()
        s0 = torch.einsum("rhd,hd->rh", q, kl[0].double().repeat_interleave(wl.g, 0)) / wl.d ** 0.5
        s5 = torch.einsum("rhd,hd->rh", q, kl[5].double().repeat_interleave(wl.g, 0)) / wl.d ** 0.5
        assert abs(s0.mean().item() - 8.0) < 0.5 and abs(s5.mean().item()) < 0.5
    assert float(k[0, 0, 0, 1]) == 0.0
    assert abs(float(k[0, 0, 0, 0]) - 8.0 * wl.d ** 0.5 / wl.SINK_QB) < 0.1


def test_normal_generator_full_mantissa_and_moments():
    """dist="normal" (bf16(N(0,1))): unit moments, tails bounded by the
    Irwin-Hall(12) support, values NOT on the 1/32 grid (full 8-bit significands), slices
    consistent, CPU generation deterministic."""
    key = TensorKey(9, "node_v", 1)
    a = bf16_tensor(key, (1 << 18,), dist="normal")
    assert torch.equal(a[1000:], bf16_tensor(key, ((1 << 18) - 1000,), offset=1000, dist="normal"))
    assert torch.equal(a, bf16_tensor(key, (1 << 18,), dist="normal"))
    x = a.double()
    assert abs(float(x.mean())) < 0.01 and abs(float(x.std()) - 1.0) < 0.01
    assert float(x.abs().max()) <= 1530 / 256
    assert float((x * 32 != (x * 32).round()).double().mean()) > 0.5
    # excess kurtosis of Irwin-Hall(12) is -0.1 (a Gaussian's is 0)
    k = float(((x - x.mean()) ** 4).mean() / x.var() ** 2) - 3
    assert -0.2 < k < 0.05


def test_scaled_workload_inputs_are_exact_power_of_two_scalings():
    """The V-range stress workload scales V by exact powers of two (node, token ramp, and the
    leaf's factor on its requests' suffix / new tokens); K and q are untouched; the per-layer
    and per-request slices equal the full tensors."""
    wl = make_config("scaled")
    base = make_config("scaled", v_scale_log2={}, v_token_scale_log2={})
    for n, p in [(0, 0), (1, 17), (2, -22), (3, 0)]:
        k, v = wl.node_kv(n, "cpu")
        kb, vb = base.node_kv(n, "cpu")
        assert torch.equal(k, kb)
        f = torch.full((v.shape[1],), 2.0 ** p, dtype=torch.float64)
        if n == 0:
            f[600:] *= 2.0 ** 20
        assert torch.equal(v.double(), vb.double() * f[None, :, None, None])
        assert torch.equal(wl.node_kv(n, "cpu", 1)[1], v[1])
    sk, sv = wl.suffix_kv("cpu")
    _, svb = base.suffix_kv("cpu")
    for r in range(0, wl.nreq, 7):
        s0, s1 = int(wl.suffix_offsets[r]), int(wl.suffix_offsets[r + 1])
        p = wl.v_scale_log2.get(wl.requests[r].leaf, 0)
        assert torch.equal(sv[:, s0:s1].double(), svb[:, s0:s1].double() * 2.0 ** p)
        assert torch.equal(wl.suffix_kv("cpu", 1, request=r)[1], sv[1, s0:s1])
        nv = wl.new_kv(0, "cpu", 1, request=r)[1]
        assert torch.equal(nv.double(), base.new_kv(0, "cpu", 1, request=r)[1].double() * 2.0 ** p)
        assert torch.equal(wl.new_kv(0, "cpu")[1][1, r], nv)
