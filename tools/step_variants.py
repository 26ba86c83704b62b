"""Device time per step of back-to-back eager fused steps (DecodePlan.run_step, one launch each, PDL-chained)
with device or pinned-host q / k / v / out -- which host-memory operand costs what (C2 shapes)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs  # noqa: E402

H, G, D, L = 8, 4, 128, 32768
dev = torch.device("cuda")
layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=16)
spec = RotationSpec(order=128, signs=make_signs(0, 0, D, 128))
R = 8
plans = []
for _ in range(R):
    t = PageTable(layout, num_pages=(L + 64) // 16 + 2, device=dev)
    t.create_sequence(0)
    sl = torch.from_numpy(t.alloc.reserve(0, L)).to(dev)
    for c0 in range(0, L, 8192):
        t.store_slots(torch.randn(8192, H, D, device=dev).bfloat16(), torch.randn(8192, H, D, device=dev).bfloat16(),
                      sl[c0:c0 + 8192], spec)
    s_np, fresh = t.alloc.plan([0])
    t._zero_pages(fresh)
    p = DecodePlan(t, [0])
    plans.append((p, torch.from_numpy(s_np).to(dev)))
torch.cuda.synchronize()
mk = {"dev": lambda x: x.to(dev), "pin": lambda x: x.pin_memory()}
q0 = torch.randn(1, H * G, D).bfloat16()
k0 = torch.randn(1, H, D).bfloat16()
v0 = torch.randn(1, H, D).bfloat16()
for qm, km, om in (("dev", "dev", "dev"), ("dev", "dev", "pin"), ("pin", "dev", "dev"), ("dev", "pin", "dev"),
                   ("pin", "pin", "pin")):
    q, k, v = mk[qm](q0), mk[km](k0), mk[km](v0)
    out = torch.empty(1, H * G, D).pin_memory() if om == "pin" else torch.empty(1, H * G, D, device=dev)
    for i in range(2 * R):
        p, s = plans[i % R]
        p.run_step(q, k, v, s, spec, out=out)
    torch.cuda.synchronize()
    n = 400
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        p, s = plans[i % R]
        p.run_step(q, k, v, s, spec, out=out)
    e1.record()
    torch.cuda.synchronize()
    print(f"q {qm} k/v {km} out {om}: {e0.elapsed_time(e1) / n * 1e3:.2f} us/step (eager, PDL-chained)")
