"""Decode-kernel error floor vs an f64 decode of the GPU's own pages, by context
length, rotation and q dtype; prints where the error concentrates.

    python tools/diag_decode.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import kvrot_oracle as O  # noqa: E402
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, Targets, make_signs  # noqa: E402


def run(L, H, G, rotate, qdtype, splits=0, kscale=1.0):
    d, P = 128, 16
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=P)
    spec = RotationSpec(order=128, signs=make_signs(0, 0, d, 128), targets=Targets.KEYS_AND_VALUES) if rotate else None
    g = torch.Generator(device="cuda").manual_seed(11)
    k = (torch.randn((L, H, d), generator=g, device="cuda") * kscale).bfloat16()
    v = torch.randn((L, H, d), generator=g, device="cuda").bfloat16()
    q = torch.randn((1, G * H, d), generator=g, device="cuda").to(qdtype)
    t = PageTable(layout, num_pages=-(-L // P))
    t.create_sequence(0)
    t.append_batch([0] * L, k, v, spec=spec, exact=True)
    plan = DecodePlan(t, [0], num_splits=splits)
    out = plan.run(q, spec)[0].double().cpu().numpy()
    kd, vd = t.read_sequence_device([0], torch.float64)
    kd, vd = kd[0].cpu().numpy(), vd[0].cpu().numpy()
    qn = q[0].double().cpu().numpy()
    qf = O.rotate_rows(qn, 128, spec.signs) if rotate else qn
    own = O.decode_flat(qf, kd, vd, G)
    if rotate:
        own = O.unrotate_rows(own, 128, spec.signs)
    err = np.abs(out - own)
    rel = err.max() / np.abs(own).max()
    # error in the stored frame (before the inverse rotation) tells QK vs PV apart
    if rotate:
        out_s = O.rotate_rows(out, 128, spec.signs) if False else None
    print(f"L={L:7d} H={H} G={G} rot={int(rotate)} q={str(qdtype)[6:]:8s} splits={plan.splits:3d} kscale={kscale}: "
          f"rel {rel:.3e}  max|ref| {np.abs(own).max():.3e}  mean|err| {err.mean():.3e}  "
          f"worst head {np.unravel_index(err.argmax(), err.shape)}", flush=True)


def main():
    for L in (16, 64, 512, 4096):
        run(L, 1, 4, False, torch.float32)
    for L in (16, 512, 4096):
        run(L, 1, 4, True, torch.float32)
        run(L, 1, 4, True, torch.bfloat16)
    run(512, 1, 8, True, torch.float32)
    run(512, 1, 1, True, torch.float32)
    run(4096, 8, 4, True, torch.float32, splits=1)
    run(4096, 8, 4, True, torch.float32, splits=4)
    run(512, 1, 4, True, torch.float32, kscale=0.1)
    run(512, 1, 4, True, torch.float32, kscale=10.0)


if __name__ == "__main__":
    main()
