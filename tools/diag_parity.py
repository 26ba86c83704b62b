"""Where does the decode error come from?  C2-sized table written by the fast K1 and by
the exact K1; each decoded and compared with (a) the oracle-quantised reference and
(b) an f64 decode of the GPU's own dequantised pages (decode-kernel error alone).
Also counts the fast K1's code / zp / scale mismatches at this size.

    python tools/diag_parity.py [L] [H] [G]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import kvrot_oracle as O  # noqa: E402
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, Targets, make_signs  # noqa: E402


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    H = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    G = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    d, P = 128, 16
    layout = HeadLayout(num_q_heads=G * H, num_kv_heads=H, head_dim=d, rot_order=128, page_tokens=P)
    spec = RotationSpec(order=128, signs=make_signs(0, 0, d, 128), targets=Targets.KEYS_AND_VALUES)
    g = torch.Generator(device="cuda").manual_seed(11)
    k = torch.randn((L, H, d), generator=g, device="cuda").bfloat16()
    v = torch.randn((L, H, d), generator=g, device="cuda").bfloat16()
    q = torch.randn((1, G * H, d), generator=g, device="cuda").bfloat16()
    kk, vv = k.double().cpu().numpy(), v.double().cpu().numpy()
    qf = O.rotate_rows(q[0].double().cpu().numpy(), 128, spec.signs)

    def store(x):
        p, s, z = O.quantize_rows(O.rotate_rows(x.reshape(-1, d), 128, spec.signs))
        return p, s, z, O.dequantize_rows(p, s, z, d).reshape(L, H, d)

    kp, ks, kz, kh = store(kk)
    vp, vs, vz, vh = store(vv)
    ref = O.unrotate_rows(O.decode_flat(qf, kh, vh, G), 128, spec.signs)
    print("max|ref|", np.abs(ref).max())
    for exact in (False, True):
        t = PageTable(layout, num_pages=L // P)
        t.create_sequence(0)
        t.append_batch([0] * L, k, v, spec=spec, exact=exact)
        out = DecodePlan(t, [0]).run(q, spec)[0].double().cpu().numpy()
        kd, vd = t.read_sequence_device([0], torch.float64)
        kd, vd = kd[0].cpu().numpy(), vd[0].cpu().numpy()
        own = O.unrotate_rows(O.decode_flat(qf, kd, vd, G), 128, spec.signs)
        e_ref = np.abs(out - ref).max() / np.abs(ref).max()
        e_own = np.abs(out - own).max() / np.abs(own).max()
        e_pages = np.abs(own - ref).max() / np.abs(ref).max()
        rec = t.page_records(t.sequence_pages(0))
        cells = P * H
        nb = cells * d // 2
        ours_kp = rec[:, :nb].reshape(-1, d // 2)
        ours_ks = rec[:, 2 * nb:2 * nb + cells * 4].copy().view(np.float32).reshape(-1)
        ours_kz = rec[:, 2 * nb + cells * 4:2 * nb + cells * 5].reshape(-1)
        x = ours_kp ^ kp
        nib = int(np.count_nonzero(x & 15) + np.count_nonzero(x & 0xF0))
        zpm = int(np.count_nonzero(ours_kz != kz))
        scm = int(np.count_nonzero(ours_ks.view(np.uint32) != ks.view(np.uint32)))
        dk = np.abs(kd - kh).max()
        print(f"exact={exact}: decode vs oracle-quantised {e_ref:.3e} | decode vs f64 of own pages {e_own:.3e} | "
              f"own pages vs oracle pages (f64 decode) {e_pages:.3e} | K nibble {nib} zp {zpm} scale {scm} "
              f"| max |k_own - k_ref| {dk:.3e}")


if __name__ == "__main__":
    main()
