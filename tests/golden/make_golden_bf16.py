"""Golden vectors for BF16 pools (cache.py:115-118, 264-266, 355-361; attention.py:67-71)
from the REAL reference implementation.  Run in the build container:

    PYTHONPATH=/root/reference/pkg/src KVROT_BACKEND=numpy python tests/golden/make_golden_bf16.py

Writes golden_bf16.npz (inputs, read_sequence outputs, decode outputs) and one
`.kvpg` dump per layout; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LAYOUTS = {"bf_small": (8, 2, 32, 32, 4), "bf_big": (32, 8, 128, 128, 16)}
LENS = (5, 17, 1)


def main() -> None:
    from kvrot.attention import DecodeRequest, decode_step
    from kvrot.cache import BF16, PageTable
    from kvrot.layout import HeadLayout
    from kvrot.rotation import RotationSpec, make_signs

    g = {}
    rng = np.random.default_rng(20261017)
    for tag, (nq, nkv, d, order, P) in LAYOUTS.items():
        layout = HeadLayout(num_q_heads=nq, num_kv_heads=nkv, head_dim=d, rot_order=order, page_tokens=P)
        spec = RotationSpec(order=order, signs=make_signs(3, 0, d, order))  # ignored by BF16 pools
        table = PageTable(layout, precision=BF16, num_pages=16)
        for s, n in enumerate(LENS):
            table.create_sequence(s)
            k = rng.standard_normal((n, nkv, d)) * 3
            v = rng.standard_normal((n, nkv, d))
            # exact bf16 rounding ties (RNE to even) and f32-subnormal inputs
            k[0, 0, :4] = [1 + 2 ** -8, 1 + 3 * 2 ** -8, -(1 + 2 ** -8), 1e-40]
            g[f"{tag}_k_{s}"], g[f"{tag}_v_{s}"] = k, v
            if s == 1:
                table.append_tokens_two_pass(s, k, v, spec=spec)
            else:
                for i in range(n):
                    table.append_token(s, k[i], v[i], spec=spec)
        for s in range(len(LENS)):
            kh, vh = table.read_sequence(s)
            g[f"{tag}_read_k_{s}"], g[f"{tag}_read_v_{s}"] = kh, vh
            q = rng.standard_normal((nq, d))
            g[f"{tag}_q_{s}"] = q
            g[f"{tag}_dec_{s}"] = decode_step(DecodeRequest(q=q, seq=s), table, spec=spec)
            g[f"{tag}_dec_nospec_{s}"] = decode_step(DecodeRequest(q=q, seq=s), table)
        table.dump(os.path.join(HERE, f"{tag}.kvpg"))
    np.savez_compressed(os.path.join(HERE, "golden_bf16.npz"), **g)
    print("wrote", len(g), "arrays")


if __name__ == "__main__":
    main()
