"""Where the e2e step's time goes (C2 shapes), on the GPU box: per-step wall time of
DecodePlan.step in a loop, with / without the host->device inputs and the
device->host output, graph replay on and off.

    python tools/e2e_probe.py [--profile]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs  # noqa: E402

H, G, D, L = 8, 4, 128, 32768
dev = torch.device("cuda")
layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=16)
spec = RotationSpec(order=128, signs=make_signs(0, 0, D, 128))
t = PageTable(layout, num_pages=(L + 20000) // 16 + 2, device=dev)
t.create_sequence(0)
sl = torch.from_numpy(t.alloc.reserve(0, L)).to(dev)
for c0 in range(0, L, 8192):
    t.store_slots(torch.randn(8192, H, D, device=dev).bfloat16(), torch.randn(8192, H, D, device=dev).bfloat16(),
                  sl[c0:c0 + 8192], spec)
kh = torch.randn(1, H, D).bfloat16().pin_memory()
vh = torch.randn(1, H, D).bfloat16().pin_memory()
qh = torch.randn(1, H * G, D).bfloat16().pin_memory()
kd, vd, qd = kh.to(dev), vh.to(dev), qh.to(dev)
oh = torch.empty(1, H * G, D).pin_memory()
od = torch.empty(1, H * G, D, device=dev)
plan = DecodePlan(t, [0], extra_tokens=16000)


def bench(name, host_in, d2h, graph, n=400, zc=True):
    """zc: the kernel writes the pinned host output itself (else device out + a D2H copy)"""
    q, k, v = (qh, kh, vh) if host_in else (qd, kd, vd)

    def one():
        if zc and d2h:  # the kernel writes the pinned host output directly
            plan.step(q, k, v, spec, out=oh, graph=graph)
            return
        plan.step(q, k, v, spec, out=od, graph=graph)
        if d2h:
            oh.copy_(od, non_blocking=True)

    for _ in range(10):
        one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        one()
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name:38s} host issue {1e6 * (t1 - t0) / n:6.1f} us/step  wall {1e6 * (t2 - t0) / n:6.1f}  "
          f"device {1e3 * e0.elapsed_time(e1) / n:6.1f}")


for side in (True, False):
  plan.side_copy = side
  print("side_copy", side)
  for zc in (True, False):
    for graph in (True, False):
        bench(f"zc={zc} host in + D2H, graph={graph}", True, True, graph, zc=zc)
        bench(f"zc={zc} host in, no D2H, graph={graph}", True, False, graph, zc=zc)
        bench(f"zc={zc} device in + D2H, graph={graph}", False, True, graph, zc=zc)
        bench(f"zc={zc} device in, no D2H, graph={graph}", False, False, graph, zc=zc)
plan.side_copy = False

if "--profile" in sys.argv:
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        plan.step(qh, kh, vh, spec, out=od, graph=True)
        oh.copy_(od, non_blocking=True)
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)

# pure host cost of one step() call (GPU drained before each call, so no back-pressure)
for graph in (True, False):
    ts = []
    for i in range(300):
        torch.cuda.synchronize()
        t0 = time.perf_counter_ns()
        plan.step(qh, kh, vh, spec, out=oh, graph=graph)
        ts.append(time.perf_counter_ns() - t0)
    ts = sorted(ts[50:])
    print(f"host latency of one step() call, graph={graph}: median {ts[len(ts) // 2] / 1e3:.1f} us, "
          f"p10 {ts[len(ts) // 10] / 1e3:.1f} us")
# pieces
plan.refresh()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
    plan.run_step(qd, kd, vd, plan.slots, spec, od)
torch.cuda.current_stream().wait_stream(s)
ts = []
for i in range(300):
    torch.cuda.synchronize()
    t0 = time.perf_counter_ns()
    g.replay()
    ts.append(time.perf_counter_ns() - t0)
ts = sorted(ts[50:])
print(f"torch CUDAGraph.replay() of one kernel node: median {ts[len(ts) // 2] / 1e3:.1f} us")
ts = []
for i in range(300):
    torch.cuda.synchronize()
    t0 = time.perf_counter_ns()
    plan.run_step(qd, kd, vd, plan.slots, spec, od)
    ts.append(time.perf_counter_ns() - t0)
ts = sorted(ts[50:])
print(f"run_step (cached ctypes args, one launch): median {ts[len(ts) // 2] / 1e3:.1f} us")
ts = []
for i in range(300):
    torch.cuda.synchronize()
    t0 = time.perf_counter_ns()
    sl_, fr_ = t.alloc.plan([0])
    ts.append(time.perf_counter_ns() - t0)
ts = sorted(ts[50:])
print(f"alloc.plan: median {ts[len(ts) // 2] / 1e3:.1f} us")


def replay_rate(g, n=400):
    for _ in range(10):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / n


print(f"back-to-back replays, device meta + device q/k/v: {replay_rate(g):.1f} us/step")
hmeta = torch.empty(16, dtype=torch.uint8).pin_memory()
hslots = hmeta[:8].view(torch.int64)
hlens = hmeta[8:12].view(torch.int32)
hslots.copy_(plan.slots.cpu())
hlens.copy_(plan.lens.cpu())
g2 = torch.cuda.CUDAGraph()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s), torch.cuda.graph(g2, stream=s):
    plan.run_step(qd, kd, vd, hslots, spec, od, lens=hlens)
torch.cuda.current_stream().wait_stream(s)
print(f"back-to-back replays, pinned-host meta: {replay_rate(g2):.1f} us/step")
g3 = torch.cuda.CUDAGraph()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s), torch.cuda.graph(g3, stream=s):
    plan.run_step(qh, kh, vh, hslots, spec, oh, lens=hlens)
torch.cuda.current_stream().wait_stream(s)
print(f"back-to-back replays, pinned-host meta + q/k/v + out: {replay_rate(g3):.1f} us/step")
