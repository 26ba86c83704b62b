"""C4-shaped decode (G = 8: 64 q / 8 kv heads, 16 sequences x 16k tokens, fused step)
for profiling the two-column-tile (NT = 2) loop.  --ncu: a few launches only."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs  # noqa: E402

B, H, G, D, L = 16, 8, int(os.environ.get("C4_G", "8")), 128, 16384
dev = torch.device("cuda")
layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=16)
spec = RotationSpec(order=128, signs=make_signs(0, 0, D, 128))
t = PageTable(layout, num_pages=B * (L // 16 + 2), device=dev)
for s in range(B):
    t.create_sequence(s)
    sl = torch.from_numpy(t.alloc.reserve(s, L)).to(dev)
    t.store_slots(torch.randn(L, H, D, device=dev).bfloat16(), torch.randn(L, H, D, device=dev).bfloat16(), sl, spec)
plan = DecodePlan(t, list(range(B)), extra_tokens=64)
q = torch.randn(B, H * G, D, device=dev).bfloat16()
kn = torch.randn(B, H, D, device=dev).bfloat16()
vn = torch.randn(B, H, D, device=dev).bfloat16()
sl, fresh = t.alloc.plan(list(range(B)))
t._zero_pages(fresh)
plan.refresh()
slots = torch.from_numpy(sl).to(dev)
n = 3 if "--ncu" in sys.argv else 50
for _ in range(n):
    plan.run_step(q, kn, vn, slots, spec)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    plan.run_step(q, kn, vn, slots, spec)
e1.record()
torch.cuda.synchronize()
us = 1e3 * e0.elapsed_time(e1) / n
byts = B * (L * 1104 + L // 16 * 4 + H * G * D * 6)
print(f"C4-shaped step (L2-warm-ish, {B}x{L}, G={G}): {us:.1f} us, {byts / us / 1e3:.0f} GB/s, splits {plan.splits}")
