"""Time the learned-R K1 (row f3) at a given token count: fused kernel vs Hadamard-only.
KVR_K1L_KAPPA_LOG2 sets the boundary margin (A/B of the exact-recomputation rate)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import HeadLayout, PageTable, RotationSpec, make_signs  # noqa: E402

n_tok = int(os.environ.get("C1_TOKENS", "65536"))
H, D, P = 8, 128, 16
dev = torch.device("cuda")
layout = HeadLayout(num_q_heads=32, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=P)
q, r = np.linalg.qr(np.random.default_rng(7).standard_normal((D, D)))
spec_h = RotationSpec(order=128, signs=make_signs(0, 0, D, 128))
spec_l = RotationSpec(order=128, signs=spec_h.signs, learned=q * np.sign(np.diag(r)), learned_values=True)
t = PageTable(layout, num_pages=n_tok // P, device=dev)
t.create_sequence(0)
t.alloc.plan([0] * n_tok)
slots = torch.arange(n_tok, dtype=torch.int64, device=dev)
g = torch.Generator(device=dev).manual_seed(1)
k = torch.randn((n_tok, H, D), generator=g, device=dev).to(torch.bfloat16)
v = torch.randn((n_tok, H, D), generator=g, device=dev).to(torch.bfloat16)


def bench(spec, n=20):
    for _ in range(3):
        t.store_slots(k, v, slots, spec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        t.store_slots(k, v, slots, spec)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


if "--ncu" in sys.argv:
    t.store_slots(k, v, slots, spec_l)
    t.store_slots(k, v, slots, spec_l)
    torch.cuda.synchronize()
    sys.exit(0)
fast = os.environ.get("KVR_K1L_FAST") == "1"
kl = os.environ.get("KVR_K1L_KAPPA_LOG2", "-20" if fast else "-18")
print(f"tokens {n_tok} mode {'fast' if fast else 'exact rows'} kappa_log2 {kl}: learned {bench(spec_l):.2f} us, "
      f"hadamard {bench(spec_h):.2f} us")
