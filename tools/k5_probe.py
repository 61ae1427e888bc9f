"""K5 (kv_scatter) throughput on the continuous-batching leg's prompt append: 32 new requests
x 255 tokens x 32 layers of K and V (1.07 GB read + written), CUDA events around
pool.append.  Usage (GPU box): python tools/k5_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2509_02121_b200 as halo  # noqa: E402
from paper_2509_02121_b200.loader import blocks_needed, load  # noqa: E402
from synth import make_config  # noqa: E402


def main():
    halo.load_library()
    wl = make_config("fanout")
    L, R, S = wl.layers, wl.nreq, wl.requests[0].suffix
    ld = load(wl, 0, capacity=blocks_needed(wl, steps=16, slack=16384))
    pool, tmpl = ld.pool, ld.node_ids[0]
    sk, sv = wl.suffix_kv("cuda:0")
    sk = sk.view(L, R, S, wl.hkv, wl.d)[:, 0].contiguous()
    sv = sv.view(L, R, S, wl.hkv, wl.d)[:, 0].contiguous()
    k = 32
    skr, svr = sk.repeat(1, k, 1, 1).contiguous(), sv.repeat(1, k, 1, 1).contiguous()
    s = torch.cuda.current_stream()
    byts = 2 * skr.numel() * 2  # K + V bytes moved (each read once, written once)
    for rep in range(6):
        reqs = [pool.open_request(tmpl) for _ in range(k)]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        pool.append(reqs, [S] * k, skr, svr)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"append {k} x {S} tokens x {L} layers: {ms * 1e3:.1f} us, {2 * byts / ms / 1e6:.0f} GB/s "
              f"(read + write)", flush=True)
        for r in reqs:
            pool.close_request(r)


if __name__ == "__main__":
    main()
