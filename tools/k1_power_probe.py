import os, sys, time, subprocess, threading
sys.path.insert(0, os.getcwd())
import torch
import paper_2509_02121_b200 as halo
from paper_2509_02121_b200.loader import append_step, load
from synth import make_config
halo.load_library()
wl = make_config("analytics", layers=2)
ld = load(wl, 0); append_step(ld, wl, 0, 0)
plan = ld.pool.plan(ld.req_ids)
q = wl.q(0, "cuda:0"); out = torch.empty((wl.nreq, wl.hq, wl.d), device="cuda:0")
samples = []
stop = False
def sampler():
    while not stop:
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown", "--format=csv,noheader,nounits"], capture_output=True, text=True)
        samples.append(r.stdout.strip()); time.sleep(0.05)
for mask, name in [(1, "K1 only"), (2, "K2 only"), (3, "K1+K2")]:
    for _ in range(20): plan.run_stages(0, mask, q[0], out)
    torch.cuda.synchronize()
    samples.clear(); stop = False
    th = threading.Thread(target=sampler); th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); n = 0; t0 = time.time()
    while time.time() - t0 < 3.0:
        for _ in range(20): plan.run_stages(0, mask, q[0], out)
        n += 20
        torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    stop = True; th.join()
    ms = e0.elapsed_time(e1) / n
    print(name, f"{ms*1e3:.1f} us/launch", samples[len(samples)//2], samples[-3:], flush=True)
