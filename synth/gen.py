"""Counter-based generator of bf16 tensors, bit-identical on CPU and CUDA.

Every element is a pure function of (seed, tensor key, flat element index), computed with
torch int64 arithmetic that never overflows, so the GPU harness can generate gigabytes
directly in HBM while a test regenerates any slice on the host for the oracle.

Value distributions (`dist`):
  "grid"   (default; round 1) an Irwin-Hall(4) approximation of a Gaussian,
               n = u0 + u1 + u2 + u3 - 126,  u_j ~ U{0..63}  (four 6-bit fields of one hash)
               x = n / 32  (exactly representable in bf16: |n| <= 126)
           so E[x] = 0, sd(x) ~= 1.155; every value is a multiple of 1/32 (products of two
           values are exact in fp32, sums of a few hundred too);
  "normal" bf16(N(0,1)) with a full mantissa (SURVEY.md §8(d) "q, k, v i.i.d. N(0,1)
           rounded to bf16"): Irwin-Hall(12) of 8-bit fields (the classic sum-of-12-uniforms
           Gaussian, tails to +-6),  x = (sum of 12 u_j - 1530) / 256,  u_j ~ U{0..255},
           sd(x) = 1.0000; x is exact in fp32 and rounded once to bf16 (round-to-nearest-
           even), so values carry all 8 significant bits and dot products round.
All integer arithmetic plus one exact scaling and one IEEE rounding: bit-identical on CPU
and GPU.  An optional power-of-two `alpha` multiplies the values exactly (the paper's
"sharpness" knob for the score distribution, SURVEY.md §8(c) error budget).

No attention arithmetic lives here ("Oracle independence").
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

_M32 = 0xFFFFFFFF
# Both multipliers are < 2**31, so (x < 2**32) * m < 2**63: no int64 overflow anywhere.
_MUL1 = 0x7FEB352D
_MUL2 = 0x5BD1E995

KINDS = {"node_k": 1, "node_v": 2, "suf_k": 3, "suf_v": 4, "q": 5, "new_k": 6, "new_v": 7}


def _hash32_int(x: int) -> int:
    x &= _M32
    x ^= x >> 16
    x = (x * _MUL1) & _M32
    x ^= x >> 15
    x = (x * _MUL2) & _M32
    x ^= x >> 16
    return x


def _hash32(x: torch.Tensor) -> torch.Tensor:
    # x: int64 tensor with values in [0, 2**32)
    x = x ^ (x >> 16)
    x = (x * _MUL1) & _M32
    x = x ^ (x >> 15)
    x = (x * _MUL2) & _M32
    x = x ^ (x >> 16)
    return x


@dataclass(frozen=True)
class TensorKey:
    seed: int
    kind: str
    ident: int

    def keys(self) -> tuple[int, int]:
        k0 = _hash32_int(self.seed * 1_000_003 + KINDS[self.kind] * 65_537 + self.ident * 7919)
        k1 = _hash32_int(k0 + 0x632BE5AB)
        return k0, k1


def bf16_tensor(key: TensorKey, shape, device="cpu", offset: int = 0, alpha: float = 1.0,
                chunk: int = 1 << 26, dist: str = "grid") -> torch.Tensor:
    """bf16 tensor of `shape` whose element i (row-major) is element offset+i of `key`."""
    shape = tuple(int(s) for s in shape)
    n = 1
    for s in shape:
        n *= s
    out = torch.empty(n, dtype=torch.bfloat16, device=device)
    k0, k1 = key.keys()
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        idx = torch.arange(offset + s, offset + e, dtype=torch.int64, device=device)
        h1 = _hash32((idx & _M32) ^ k0)
        h2 = _hash32(h1 ^ ((idx >> 32) & _M32) ^ k1)
        if dist == "grid":
            tot = (h2 & 63) + ((h2 >> 8) & 63) + ((h2 >> 16) & 63) + ((h2 >> 24) & 63) - 126
            out[s:e] = (tot.to(torch.float32) * (alpha / 32.0)).to(torch.bfloat16)
        elif dist == "normal":
            h3 = _hash32(h2 ^ k0 ^ 0x9E3779B9)
            h4 = _hash32(h3 ^ k1 ^ 0x7F4A7C15)
            tot = -1530
            for h in (h2, h3, h4):
                tot = tot + (h & 255) + ((h >> 8) & 255) + ((h >> 16) & 255) + ((h >> 24) & 255)
            out[s:e] = (tot.to(torch.float32) * (alpha / 256.0)).to(torch.bfloat16)
        else:
            raise ValueError(f"unknown dist {dist!r}")
    return out.view(shape)


def bf16_bits(t: torch.Tensor) -> np.ndarray:
    """bf16 tensor -> numpy uint16 bit patterns (host copy)."""
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns to float64 (bf16 is the top half of an fp32)."""
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
