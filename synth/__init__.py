"""Seeded synthetic workloads shared by the oracle tests, the CUDA parity tests and bench.py.

This package holds NO attention arithmetic: only a counter-based integer generator that
produces bf16 bit patterns, and the shapes of the paper's workloads (prefix trees of
template fan-out, Llama-3-8B GQA heads).  Both the oracle side and the CUDA side import
it; neither imports the other.
"""
from .gen import bf16_tensor, bf16_to_f64, TensorKey
from .workloads import Workload, NodeSpec, RequestSpec, make_config, CONFIGS

__all__ = ["bf16_tensor", "bf16_to_f64", "TensorKey", "Workload", "NodeSpec",
           "RequestSpec", "make_config", "CONFIGS"]
