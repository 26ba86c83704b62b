"""Soak test of the serving step (GPU box): many DecodePlan.step calls through the native step
ring with pinned host inputs / output, crossing page boundaries (general path every 16th step),
with periodic NaN injections (rejected, nothing committed) and periodic full checks of the
output against a fresh decode of the same table state (decode_batch, no ring, no graph).

    python tools/soak_step.py [steps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs  # noqa: E402
from paper_2604_19157_b200.attention import decode_batch  # noqa: E402
from paper_2604_19157_b200.errors import NonFiniteInputError  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
EVERY = int(os.environ.get("SOAK_EVERY", "500"))  # steps between full checks
B, H, D = 3, 8, 128
G = int(os.environ.get("SOAK_G", "4"))
P = int(os.environ.get("SOAK_P", "16"))
dev = torch.device("cuda")
layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=P)
from paper_2604_19157_b200 import Targets  # noqa: E402
spec = RotationSpec(order=128, signs=make_signs(1, 0, D, 128),
                    targets=Targets.KEYS_ONLY if os.environ.get("SOAK_KEYS_ONLY") else Targets.KEYS_AND_VALUES)
if os.environ.get("SOAK_LEARNED"):  # row f3: a learned R (unfused exact write + row-matmul query / output)
    _q, _r = np.linalg.qr(np.random.default_rng(3).standard_normal((D, D)))
    spec = RotationSpec(order=128, signs=spec.signs, learned=_q * np.sign(np.diag(_r)), learned_values=True)
prec = "bf16" if os.environ.get("SOAK_BF16") else "int4"
t = PageTable(layout, precision=prec, num_pages=(B * (2000 + N // 1)) // P + 16, device=dev)
rng = np.random.default_rng(0)
for s in range(B):
    t.create_sequence(s)
    L0 = 500 + 700 * s
    t.append_batch([s] * L0, torch.randn(L0, H, D, device=dev).bfloat16(), torch.randn(L0, H, D, device=dev).bfloat16(),
                   spec=spec, check=False)
plan = DecodePlan(t, list(range(B)), extra_tokens=N + 32)
qh = torch.empty(B, H * G, D, dtype=torch.bfloat16).pin_memory()
kh = torch.empty(B, H, D, dtype=torch.bfloat16).pin_memory()
vh = torch.empty(B, H, D, dtype=torch.bfloat16).pin_memory()
oh = torch.empty(B, H * G, D).pin_memory()
worst = 0.0
rejected = checks = 0
for i in range(N):
    qh.copy_(torch.randn(B, H * G, D).bfloat16())
    kh.copy_(torch.randn(B, H, D).bfloat16())
    vh.copy_(torch.randn(B, H, D).bfloat16())
    if i % 997 == 13:  # a NaN: rejected before anything is committed
        kh[1, 3, 7] = float("nan")
        lens0 = [t.sequence_length(s) for s in range(B)]
        try:
            plan.step(qh, kh, vh, spec, out=oh, graph=True)
            raise AssertionError("NaN input was accepted")
        except NonFiniteInputError:
            rejected += 1
        assert [t.sequence_length(s) for s in range(B)] == lens0
        continue
    plan.step(qh, kh, vh, spec, out=oh, graph=True)
    if i % EVERY == EVERY - 1:
        torch.cuda.synchronize()
        ref = decode_batch(qh.cuda().float(), t, list(range(B)), spec=spec).cpu()
        err = float((oh - ref).abs().max() / ref.abs().max())
        worst = max(worst, err)
        checks += 1
        assert err < 1e-5, (i, err)
torch.cuda.synchronize()
t.check_flags()
print(f"soak: {N} steps, {rejected} NaN steps rejected, {checks} checks against a fresh decode, "
      f"max rel diff {worst:.2e}, lengths {[t.sequence_length(s) for s in range(B)]}")
