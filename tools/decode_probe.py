"""One decode configuration for ncu / A/B: B sequences x L tokens, 8 kv heads, G q heads per kv head.

    python tools/decode_probe.py B L G [--fused] [--ncu]
Prints the per-launch time over rotating tables (> 2x L2); --ncu runs a few launches only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs  # noqa: E402

B, L, G = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
SPL = [int(a[len("--splits="):]) for a in sys.argv if a.startswith("--splits=")]
SPL = SPL[0] if SPL else 0
H, D, P = 8, 128, 16
dev = torch.device("cuda")
layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=P)
spec = RotationSpec(order=128, signs=make_signs(0, 0, D, 128))
g = torch.Generator(device=dev).manual_seed(3)
per_table = B * L * H * 138
reps = max(1, min(8, -(-300_000_000 // per_table)))
plans, qs = [], []
for rr in range(reps):
    t = PageTable(layout, num_pages=B * (L // P + 1), device=dev)
    for b in range(B):
        t.create_sequence(b)
        sl = torch.from_numpy(t.alloc.reserve(b, L)).to(dev)
        for c0 in range(0, L, 16384):
            n = min(16384, L - c0)
            t.store_slots(torch.randn((n, H, D), generator=g, device=dev).bfloat16(),
                          torch.randn((n, H, D), generator=g, device=dev).bfloat16(), sl[c0:c0 + n], spec)
    plans.append(DecodePlan(t, list(range(B)), num_splits=SPL))
    qs.append(torch.randn((B, H * G, D), generator=g, device=dev).bfloat16())
torch.cuda.synchronize()
n = 4 if "--ncu" in sys.argv else 200
for i in range(3):
    plans[i % reps].run(qs[i % reps], spec)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(n):
    plans[i % reps].run(qs[i % reps], spec)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / n * 1e3
print(f"B {B} L {L} G {G} splits {plans[0].splits}: {us:.2f} us/launch, {B * L * H * 138 / (us * 1e-6) / 1e9:.0f} GB/s")
