"""Serving soak (GPU box): decode steps for B sequences through DecodePlan.step (device or pinned
host inputs), interleaved on the same stream with bulk prefill writes (append_batch, K1) into
another sequence and with decodes of that sequence (decode_batch), outputs checked against fresh
decodes of the same table state.  Exercises the pool-write notes that gate the decode's pre-wait
reads after a K1 write, page allocation, graph replay and the step ring together.

    python tools/soak_serving.py [steps] [--device]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs  # noqa: E402
from paper_2604_19157_b200.attention import decode_batch  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else 4000
DEVICE = "--device" in sys.argv
B, H, G, D = 2, 8, 4, 128
dev = torch.device("cuda")
layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=16)
spec = RotationSpec(order=128, signs=make_signs(3, 1, D, 128))
t = PageTable(layout, num_pages=(B * (3000 + N) + 4 * N * 8) // 16 + 64, device=dev)
torch.manual_seed(1)
for s in range(B):
    t.create_sequence(s)
    L0 = 800 + 900 * s
    t.append_batch([s] * L0, torch.randn(L0, H, D, device=dev).bfloat16(), torch.randn(L0, H, D, device=dev).bfloat16(),
                   spec=spec, check=False)
PRE = 100  # the prefilled sequence
t.create_sequence(PRE)
plan = DecodePlan(t, list(range(B)), extra_tokens=N + 32)
if DEVICE:
    q = torch.empty(B, H * G, D, dtype=torch.bfloat16, device=dev)
    k = torch.empty(B, H, D, dtype=torch.bfloat16, device=dev)
    v = torch.empty(B, H, D, dtype=torch.bfloat16, device=dev)
    out = torch.empty(B, H * G, D, device=dev)
else:
    q = torch.empty(B, H * G, D, dtype=torch.bfloat16).pin_memory()
    k = torch.empty(B, H, D, dtype=torch.bfloat16).pin_memory()
    v = torch.empty(B, H, D, dtype=torch.bfloat16).pin_memory()
    out = torch.empty(B, H * G, D).pin_memory()
worst = worst_pre = 0.0
checks = 0
for i in range(N):
    q.copy_(torch.randn(B, H * G, D, device=dev).bfloat16())
    k.copy_(torch.randn(B, H, D, device=dev).bfloat16())
    v.copy_(torch.randn(B, H, D, device=dev).bfloat16())
    plan.step(q, k, v, spec, out=out, graph=True, check=not DEVICE)
    if i % 7 == 3:  # a prefill chunk of another sequence right behind the step, then its decode
        n = 64 + (i % 5) * 48
        t.append_batch([PRE] * n, torch.randn(n, H, D, device=dev).bfloat16(),
                       torch.randn(n, H, D, device=dev).bfloat16(), spec=spec, check=False)
        qp = torch.randn(1, H * G, D, device=dev)
        op = decode_batch(qp, t, [PRE], spec=spec)
    if i % 50 == 49:
        torch.cuda.synchronize()
        ref = decode_batch(q.float().cuda(), t, list(range(B)), spec=spec).cpu()
        err = float((out.cpu() - ref).abs().max() / ref.abs().max())
        worst = max(worst, err)
        ref_p = decode_batch(qp, t, [PRE], spec=spec)  # the same table state: must be identical
        worst_pre = max(worst_pre, float((op - ref_p).abs().max()))
        checks += 1
        assert err < 1e-5, (i, err)
torch.cuda.synchronize()
t.check_flags()
print(f"serving soak ({'device' if DEVICE else 'pinned host'} inputs): {N} steps, {checks} checks, "
      f"max rel diff {worst:.2e}, prefill-decode replay diff {worst_pre:.1e}, "
      f"lengths {[t.sequence_length(s) for s in range(B)]} + {t.sequence_length(PRE)}")
