"""Where does the end-to-end step time go?  (GPU box; diagnostics, not product.)
Times 20 C1 decode steps through halo_decode_step with device buffers vs pinned host
buffers, wall clock and CUDA events, and the host time spent inside the API calls."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2509_02121_b200 as halo  # noqa: E402
from paper_2509_02121_b200.loader import blocks_needed, load  # noqa: E402
from synth import make_config  # noqa: E402


def main():
    wl = make_config("fanout")
    ld = load(wl, 0, capacity=blocks_needed(wl, steps=2, slack=4096))
    pool, reqs = ld.pool, ld.req_ids
    L, R, Hq, D = wl.layers, wl.nreq, wl.hq, wl.d
    nk, nv = wl.new_kv(0, "cuda")
    q = wl.q(0, "cuda")
    out = torch.empty((L, R, Hq, D), device="cuda")
    ones = [1] * R
    pool.append(reqs, ones, nk, nv)
    plan = pool.plan(reqs)
    hk, hv, hq = nk.cpu().pin_memory(), nv.cpu().pin_memory(), q.cpu().pin_memory()
    ho = torch.empty((L, R, Hq, D), pin_memory=True)
    for name, args in [("device", (nk, nv, q, out)), ("host", (hk, hv, hq, ho)),
                       ("host-in dev-out", (hk, hv, hq, out)), ("dev-in host-out", (nk, nv, q, ho))]:
        for _ in range(3):
            pool.truncate(reqs, ones)
            pool.decode_step(reqs, *args, reuse=plan)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        api = 0.0
        t0 = time.perf_counter()
        e0.record()
        for _ in range(n):
            a = time.perf_counter()
            pool.truncate(reqs, ones)
            pool.decode_step(reqs, *args, reuse=plan)
            api += time.perf_counter() - a
        e1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        print(f"{name:16s} wall {wall / n * 1e3:7.3f} ms/step  events {e0.elapsed_time(e1) / n:7.3f} ms/step  "
              f"host in API {api / n * 1e3:7.3f} ms/step  -> {R * L / (wall / n) / 1e6:.3f} M q/s", flush=True)
    # raw copy rates
    for nbytes in (100 << 20, 134 << 20):
        h = torch.empty(nbytes // 4, pin_memory=True)
        d = torch.empty(nbytes // 4, device="cuda")
        for direction in ("h2d", "d2h"):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(5):
                (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / 5
            print(f"{direction} {nbytes >> 20} MiB: {nbytes / dt / 1e9:.1f} GB/s")
    # both directions at once (two streams): is PCIe full duplex here?
    hi, di = torch.empty((100 << 20) // 4, pin_memory=True), torch.empty((100 << 20) // 4, device="cuda")
    ho2, do2 = torch.empty((134 << 20) // 4, pin_memory=True), torch.empty((134 << 20) // 4, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1):
            di.copy_(hi, non_blocking=True)
        with torch.cuda.stream(s2):
            ho2.copy_(do2, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"concurrent h2d 100 MiB + d2h 134 MiB: {dt * 1e3:.2f} ms ({234 * 1.048576 / dt / 1e3:.1f} GB/s total)")
    plan.destroy()
    pool.destroy()


if __name__ == "__main__":
    main()
