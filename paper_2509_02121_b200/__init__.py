"""B200-native shared-prefix decode attention (the data path behind Halo's KV-cache
sharing, arXiv 2509.02121).

This module is a thin ctypes binding over the C-ABI library libhalo_attn.so
(include/halo_attn.h): argument marshalling only.  Every step of the hot path runs in the
library's CUDA kernels; there is no CPU fallback -- importing this package without the
built library raises.  torch is used only for device memory and streams.
"""
from .abi import (HaloError, Pool, Plan, PlanOptions, lib_path, load_library, comm_unique_id,
                  place_groups, STATUS)

__all__ = ["HaloError", "Pool", "Plan", "PlanOptions", "lib_path", "load_library",
           "comm_unique_id", "place_groups", "STATUS"]
