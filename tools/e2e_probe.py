"""Host-side cost of DecodePlan.step (C2 shapes) broken down, on the GPU box."""
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
t = PageTable(layout, num_pages=(L + 4096) // 16 + 2, device=dev)
t.create_sequence(0)
sl = torch.from_numpy(t.alloc.reserve(0, L)).to(dev)
for c0 in range(0, L, 8192):
    t.store_slots(torch.randn(8192, H, D, device=dev).bfloat16(), torch.randn(8192, H, D, device=dev).bfloat16(),
                  sl[c0:c0 + 8192], spec)
kh = torch.randn(1, H, D).bfloat16().pin_memory()
vh = torch.randn(1, H, D).bfloat16().pin_memory()
qh = torch.randn(1, H * G, D).bfloat16().pin_memory()
oh = torch.empty(1, H * G, D).pin_memory()
od = torch.empty(1, H * G, D, device=dev)
plan = DecodePlan(t, [0], extra_tokens=4000)
GRAPH = "--graph" in sys.argv
for _ in range(20):
    plan.step(qh, kh, vh, spec, out=od, graph=GRAPH)
    oh.copy_(od, non_blocking=True)
torch.cuda.synchronize()
N = 500
t0 = time.perf_counter()
for _ in range(N):
    plan.step(qh, kh, vh, spec, out=od, graph=GRAPH)
    oh.copy_(od, non_blocking=True)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue {1e6 * (t1 - t0) / N:.1f} us/step, wall incl. drain {1e6 * (t2 - t0) / N:.1f} us/step")
import cProfile
import pstats
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    plan.step(qh, kh, vh, spec, out=od, graph=GRAPH)
    oh.copy_(od, non_blocking=True)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
