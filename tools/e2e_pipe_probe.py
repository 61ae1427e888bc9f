"""Pipeline-shape probe for the end-to-end decode step (GPU box; diagnostics only).
Mimics halo_decode_step's per-layer copy/compute overlap with torch streams around the
real K5/K1/K2 launches, for several copy orderings, and reports ms/step."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2509_02121_b200.loader import blocks_needed, load  # noqa: E402
from synth import make_config  # noqa: E402


def main():
    wl = make_config("fanout")
    ld = load(wl, 0, capacity=blocks_needed(wl, steps=2, slack=4096))
    pool, reqs = ld.pool, ld.req_ids
    L, R, Hq, Hkv, D = wl.layers, wl.nreq, wl.hq, wl.hkv, wl.d
    nk, nv = wl.new_kv(0, "cuda")
    q = wl.q(0, "cuda")
    out = torch.empty((L, R, Hq, D), device="cuda")
    ones = [1] * R
    pool.append(reqs, ones, nk, nv)
    plan = pool.plan(reqs)
    hk, hv, hq = nk.cpu().pin_memory(), nv.cpu().pin_memory(), q.cpu().pin_memory()
    ho = torch.empty((L, R, Hq, D), pin_memory=True)
    dk, dv, dq = torch.empty_like(nk), torch.empty_like(nv), torch.empty_like(q)
    s = torch.cuda.current_stream()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(L)]
    ev_out = [torch.cuda.Event() for _ in range(L)]

    def step(mode):
        start = torch.cuda.Event()
        start.record(s)
        sa.wait_event(start)
        sb.wait_event(start)
        if mode in ("upfront", "upfront-noout"):
            with torch.cuda.stream(sa):
                for l in range(L):
                    dk[l].copy_(hk[l], non_blocking=True)
                    dv[l].copy_(hv[l], non_blocking=True)
                    dq[l].copy_(hq[l], non_blocking=True)
                    ev_in[l].record(sa)
        if mode.startswith("h"):  # hXdYpZ: H2D in X-layer chunks at most Z chunks ahead of
            import re                # compute (0: all upfront), D2H in Y-layer chunks
            X, Y, Z = map(int, re.match(r"h(\d+)d(\d+)p(\d+)", mode).groups())
            nch = (L + X - 1) // X
            ev_started = [torch.cuda.Event() for _ in range(nch)]

            def h2d(c):
                c0 = c * X
                with torch.cuda.stream(sa):
                    if Z > 0 and c - Z >= 0:
                        sa.wait_event(ev_started[c - Z])
                    dk[c0:c0 + X].copy_(hk[c0:c0 + X], non_blocking=True)
                    dv[c0:c0 + X].copy_(hv[c0:c0 + X], non_blocking=True)
                    dq[c0:c0 + X].copy_(hq[c0:c0 + X], non_blocking=True)
                    ev_in[c0].record(sa)
            for c in range(nch if Z == 0 else min(Z, nch)):
                h2d(c)
            for l in range(L):
                if l % X == 0:
                    s.wait_event(ev_in[l])
                    c = l // X
                    ev_started[c].record(s)
                    if Z > 0 and c + Z < nch:
                        h2d(c + Z)
                plan.run(l, dq[l], out[l])
                if l % Y == Y - 1 or l == L - 1:
                    ev_out[l].record(s)
                    c0 = l - l % Y
                    with torch.cuda.stream(sb):
                        sb.wait_event(ev_out[l])
                        ho[c0:l + 1].copy_(out[c0:l + 1], non_blocking=True)
            done = torch.cuda.Event()
            done.record(sb)
            s.wait_event(done)
            return
        if mode.startswith("chunk"):  # copies grouped G layers at a time, both directions
            G = int(mode[5:])
            with torch.cuda.stream(sa):
                for c0 in range(0, L, G):
                    dk[c0:c0 + G].copy_(hk[c0:c0 + G], non_blocking=True)
                    dv[c0:c0 + G].copy_(hv[c0:c0 + G], non_blocking=True)
                    dq[c0:c0 + G].copy_(hq[c0:c0 + G], non_blocking=True)
                    ev_in[c0].record(sa)
            for l in range(L):
                if l % G == 0:
                    s.wait_event(ev_in[l])
                plan.run(l, dq[l], out[l])
                if l % G == G - 1 or l == L - 1:
                    ev_out[l].record(s)
                    c0 = l - l % G
                    with torch.cuda.stream(sb):
                        sb.wait_event(ev_out[l])
                        ho[c0:l + 1].copy_(out[c0:l + 1], non_blocking=True)
            done = torch.cuda.Event()
            done.record(sb)
            s.wait_event(done)
            return
        for l in range(L):
            if mode == "jit":
                with torch.cuda.stream(sa):
                    if l == 0:
                        for j in range(2):
                            dk[j].copy_(hk[j], non_blocking=True)
                            dv[j].copy_(hv[j], non_blocking=True)
                            dq[j].copy_(hq[j], non_blocking=True)
                            ev_in[j].record(sa)
                    if l + 2 < L:
                        sa.wait_event(ev_out[l - 1] if l >= 1 else start)
                        j = l + 2
                        dk[j].copy_(hk[j], non_blocking=True)
                        dv[j].copy_(hv[j], non_blocking=True)
                        dq[j].copy_(hq[j], non_blocking=True)
                        ev_in[j].record(sa)
            if mode != "none":
                s.wait_event(ev_in[l])
            plan.run(l, dq[l] if mode != "none" else q[l], out[l])
            ev_out[l].record(s)
            if mode in ("upfront", "jit", "outonly"):
                with torch.cuda.stream(sb):
                    sb.wait_event(ev_out[l])
                    ho[l].copy_(out[l], non_blocking=True)
        done = torch.cuda.Event()
        done.record(sb)
        s.wait_event(done)

    modes = sys.argv[1:] or ["none", "outonly", "upfront-noout", "upfront", "jit", "chunk2", "chunk4", "chunk8"]
    for mode in modes:
        for _ in range(3):
            step(mode)
        torch.cuda.synchronize()
        n = 15
        t0 = time.perf_counter()
        for _ in range(n):
            step(mode)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / n
        print(f"{mode:14s} {dt * 1e3:7.3f} ms/step  {R * L / dt / 1e6:.3f} M q/s", flush=True)


if __name__ == "__main__":
    main()
