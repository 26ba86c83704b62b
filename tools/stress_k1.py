"""Randomised K1 stress (GPU box): random token counts across both kernels' dispatch range, random
slot permutations, head counts, orders, targets and row families; the fast bf16 write must give the
exact (f64) path's codes and zero points bit for bit and scales within 2 f32 ulp.

    python tools/stress_k1.py [cases]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import HeadLayout, PageTable, RotationSpec, Targets, make_signs  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from kvtest_util import bf16_round, gen_rows  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rng = np.random.default_rng(11)
dev = torch.device("cuda")
worst_ulp = 0
for c in range(cases):
    H = int(rng.choice([1, 2, 4, 8]))
    P = int(rng.choice([16, 32, 64]))
    order = int(rng.choice([16, 32, 64, 128]))
    n = int(rng.choice([1, 7, 100, 1000, 5000, 20000, 40000, 80000])) + int(rng.integers(0, 50))
    kind = str(rng.choice(["gaussian", "outlier", "correlated", "adversarial"]))
    targets = Targets.KEYS_ONLY if rng.random() < 0.3 else Targets.KEYS_AND_VALUES
    rotate = rng.random() < 0.85
    layout = HeadLayout(num_q_heads=4 * H, num_kv_heads=H, head_dim=128, rot_order=order, page_tokens=P)
    spec = RotationSpec(order=order, signs=make_signs(int(rng.integers(0, 99)), 0, 128, order), targets=targets) \
        if rotate else None
    pages = n // P + 2
    perm = torch.from_numpy(rng.permutation(pages * P)[:n].astype(np.int64)).to(dev)
    k = torch.tensor(bf16_round(gen_rows(kind, n * H, 128, c)).reshape(n, H, 128)).to(torch.bfloat16).to(dev)
    v = torch.tensor(bf16_round(gen_rows(kind, n * H, 128, c + 1000)).reshape(n, H, 128)).to(torch.bfloat16).to(dev)
    ta = PageTable(layout, num_pages=pages, device=dev)
    tb = PageTable(layout, num_pages=pages, device=dev)
    ta.store_slots(k, v, perm, spec)
    tb.store_slots(k, v, perm, spec, exact=True)
    torch.cuda.synchronize()
    a = ta.pool.view(pages, -1).cpu().numpy()
    b = tb.pool.view(pages, -1).cpu().numpy()
    # cell layout: k_scale f32[16] | v_scale f32[16] | codes (2 x 1024) | zp (2 x 16) per 2208-B cell
    cells_a = a.reshape(-1, 2208)
    cells_b = b.reshape(-1, 2208)
    codes_eq = np.array_equal(cells_a[:, 128:2208], cells_b[:, 128:2208])
    sa = cells_a[:, :128].copy().view(np.int32)
    sb = cells_b[:, :128].copy().view(np.int32)
    ulp = int(np.abs(sa.astype(np.int64) - sb.astype(np.int64)).max())
    worst_ulp = max(worst_ulp, ulp)
    print(f"case {c}: n={n} H={H} P={P} order={order} {kind} {targets.name if rotate else 'plain'}: "
          f"codes+zp equal {codes_eq}, scale ulp {ulp}")
    assert codes_eq, c
    assert ulp <= 2, c
print(f"stress_k1: {cases} cases, codes / zero points bit-exact, worst scale {worst_ulp} ulp")
