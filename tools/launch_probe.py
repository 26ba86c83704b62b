"""Device time per fused step for different launch styles (C2 shapes, device inputs):
eager back-to-back kvr_decode_step launches (PDL-chained), one CUDA graph of many steps,
and one graph launch per step."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs  # noqa: E402

H, G, D, L = 8, 4, 128, int(os.environ.get("CTX", "32768"))
dev = torch.device("cuda")
layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=16)
spec = RotationSpec(order=128, signs=make_signs(0, 0, D, 128))
t = PageTable(layout, num_pages=(L + 64) // 16 + 2, device=dev)
t.create_sequence(0)
sl = torch.from_numpy(t.alloc.reserve(0, L)).to(dev)
for c0 in range(0, L, 8192):
    n = min(8192, L - c0)
    t.store_slots(torch.randn(n, H, D, device=dev).bfloat16(), torch.randn(n, H, D, device=dev).bfloat16(),
                  sl[c0:c0 + n], spec)
slot, _ = t.alloc.plan([0])
slot = torch.from_numpy(slot).to(dev)
plan = DecodePlan(t, [0])
q = torch.randn(1, H * G, D, device=dev).bfloat16()
kn = torch.randn(1, H, D, device=dev).bfloat16()
vn = torch.randn(1, H, D, device=dev).bfloat16()
out = torch.empty(1, H * G, D, device=dev)
pin_out = torch.empty(1, H * G, D).pin_memory()


def one(o=out):
    plan.run_step(q, kn, vn, slot, spec, o)


for _ in range(20):
    one()
torch.cuda.synchronize()
N = 2000
for name, o in (("eager launches, device out", out), ("eager launches, pinned host out", pin_out)):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(N):
        one(o)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / N * 1e3:.2f} us/step device, {(time.perf_counter() - t0) / N * 1e6:.2f} wall")
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
    for _ in range(64):
        one()
torch.cuda.current_stream().wait_stream(s)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(16):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"one graph of 64 steps: {e0.elapsed_time(e1) / 1024 * 1e3:.2f} us/step")
g1 = torch.cuda.CUDAGraph()
with torch.cuda.stream(s), torch.cuda.graph(g1, stream=s):
    one()
torch.cuda.current_stream().wait_stream(s)
g1.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(N):
    g1.replay()
e1.record()
torch.cuda.synchronize()
print(f"one graph launch per step: {e0.elapsed_time(e1) / N * 1e3:.2f} us/step")

# ring-like variants: an event record after every step; slot ids / lengths in pinned host memory
from paper_2604_19157_b200 import _kernels  # noqa: E402
evs = [_kernels.host_event() for _ in range(4)]
stream = torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())
slot_pin = slot.cpu().pin_memory()
lens_pin = plan.lens.cpu().pin_memory()
variants = {
    "eager + event record per step": lambda i: (one(), _kernels.event_record(evs[i % 4], stream)),
    "eager, slot/len pinned": lambda i: plan.run_step(q, kn, vn, slot_pin, spec, out, lens=lens_pin),
    "eager, slot/len pinned + event": lambda i: (plan.run_step(q, kn, vn, slot_pin, spec, out, lens=lens_pin),
                                                 _kernels.event_record(evs[i % 4], stream)),
}
for name, fn in variants.items():
    for i in range(20):
        fn(i)
    torch.cuda.synchronize()
    e0.record()
    for i in range(N):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / N * 1e3:.2f} us/step")
