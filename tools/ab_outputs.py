"""Decode outputs of the in-tree library for a fixed input, saved for an A/B
bit-identity check between two library builds (KVR_LIB_PATH selects one).

    python tools/ab_outputs.py OUT.pt"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs  # noqa: E402

outs = []
for H, G, L, B in ((8, 4, 32768, 1), (8, 4, 3000, 3), (1, 4, 200000, 1), (8, 8, 5000, 2)):
    gen = torch.Generator(device="cuda").manual_seed(7)
    layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=128, rot_order=128, page_tokens=16)
    spec = RotationSpec(order=128, signs=make_signs(1, 0, 128, 128))
    t = PageTable(layout, num_pages=B * (L // 16 + 4), device="cuda")
    for s in range(B):
        t.create_sequence(s)
        sl = torch.from_numpy(t.alloc.reserve(s, L - 7 * s)).cuda()
        n = L - 7 * s
        t.store_slots(torch.randn(n, H, 128, generator=gen, device="cuda").bfloat16(),
                      torch.randn(n, H, 128, generator=gen, device="cuda").bfloat16(), sl, spec)
    q = torch.randn(B, H * G, 128, generator=gen, device="cuda").bfloat16()
    plan = DecodePlan(t, list(range(B)), extra_tokens=1)
    outs.append(plan.run(q, spec).cpu())
    kn = torch.randn(B, H, 128, generator=gen, device="cuda").bfloat16()
    vn = torch.randn(B, H, 128, generator=gen, device="cuda").bfloat16()
    outs.append(plan.step(q, kn, vn, spec).cpu())
torch.save(outs, sys.argv[1])
print("saved", len(outs))
