"""Randomised decode stress (GPU box): random batch / lengths (ragged, incl. 1 and page-aligned),
head counts, GQA group sizes, page sizes, orders, targets and split counts; the INT4 decode kernel
against the flat f64 decode of the same dequantised pages (kvr_decode_flat_f64), within 1e-5 of
max|ref|.

    python tools/stress_decode.py [cases]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, Targets, make_signs  # noqa: E402
from paper_2604_19157_b200.attention import decode_step_fp  # noqa: E402
from paper_2604_19157_b200.rotation import apply_block_rotation, apply_inverse_rotation, value_branch_spec  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rng = np.random.default_rng(5)
dev = torch.device("cuda")
worst = 0.0
for c in range(cases):
    H = int(rng.choice([1, 2, 4, 8]))
    G = int(rng.choice([1, 2, 4, 8]))
    P = int(rng.choice([16, 32, 64]))
    order = int(rng.choice([16, 32, 64, 128]))
    B = int(rng.integers(1, 6))
    lens = [int(rng.choice([1, 15, 16, 17, int(rng.integers(2, 5000)), int(rng.integers(5000, 40000))])) for _ in range(B)]
    targets = Targets.KEYS_ONLY if rng.random() < 0.3 else Targets.KEYS_AND_VALUES
    spec = RotationSpec(order=order, signs=make_signs(int(rng.integers(0, 99)), 0, 128, order), targets=targets)
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=128, rot_order=order, page_tokens=P)
    t = PageTable(layout, num_pages=sum(L // P + 1 for L in lens) + 2, device=dev)
    for s, L in enumerate(lens):
        t.create_sequence(s)
        t.append_batch([s] * L, torch.randn(L, H, 128, device=dev).bfloat16(), torch.randn(L, H, 128, device=dev).bfloat16(),
                       spec=spec, check=False)
    splits = int(rng.choice([0, 0, 1, 3, 8, 12, 40]))
    plan = DecodePlan(t, list(range(B)), num_splits=splits)
    q = torch.randn(B, G * H, 128, device=dev)
    out = plan.run(q, spec).cpu().numpy()
    kd, vd = t.read_sequence_device(list(range(B)), torch.float64)
    vspec = value_branch_spec(spec)
    err = 0.0
    for b, L in enumerate(lens):
        qr = apply_block_rotation(q[b].double(), layout, spec).cpu().numpy()
        o = decode_step_fp(qr, kd[b, :L].cpu().numpy(), vd[b, :L].cpu().numpy(), layout)
        if vspec is not None:
            o = apply_inverse_rotation(torch.tensor(o).cuda(), layout, vspec).cpu().numpy()
        err = max(err, float(np.abs(out[b] - o).max() / np.abs(o).max()))
    worst = max(worst, err)
    print(f"case {c}: B={B} lens={lens} H={H} G={G} P={P} order={order} {targets.name} splits={plan.splits}: {err:.2e}")
    assert err <= 1e-5, c
print(f"stress_decode: {cases} cases, worst rel err {worst:.2e}")
