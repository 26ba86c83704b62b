"""Generate golden vectors from the REAL reference implementation.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src KVROT_BACKEND=numpy \
        python tests/golden/make_golden.py

It imports `kvrot` read-only and writes small fixtures next to this script:
  golden_v1.npz      -- kernel / rotation / quantization / decode vectors
  *.kvpg             -- page-table dumps produced by kvrot.cache.PageTable.dump

The fixtures pin both the numpy oracle (oracle/kvrot_oracle.py) and the CUDA
product path; nothing at test or bench time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def bf16_exact(a: np.ndarray) -> np.ndarray:
    """Round f64 values to the nearest bf16 (RNE via f32), returned as f64."""
    from kvrot.cache import bf16_bits_to_float, float_to_bf16_bits

    return bf16_bits_to_float(float_to_bf16_bits(np.asarray(a, dtype=np.float64))).reshape(np.shape(a))


def main() -> None:
    import kvrot
    from kvrot import _kernels
    from kvrot.attention import DecodeRequest, decode_step, decode_step_fp
    from kvrot.cache import INT4, PageTable
    from kvrot.harness import default_correlated_spec, default_outlier_spec, generate_kv
    from kvrot.layout import HeadLayout
    from kvrot.rotation import RotationSpec, Targets, apply_block_rotation, apply_inverse_rotation, make_signs

    assert _kernels.get_backend() == "numpy", "generate goldens with KVROT_BACKEND=numpy"
    g = {}
    rng = np.random.default_rng(20261017)

    # --- fwht_rows (_ref.py:22-40), incl. adversarial magnitudes (test_kernels.py:69-95)
    x = rng.standard_normal((37, 256)) * 50
    g["fwht_in"] = x
    for order in (1, 2, 4, 16, 32, 64, 128):
        y = x.copy()
        _kernels.fwht_rows(y, order)
        g[f"fwht_out_{order}"] = y
    adv = np.array([[1e-300, -1e300, 3.0, -3.0, 1e16, 1.0, -1e-16, 0.0] * 16])
    g["fwht_adv_in"] = adv
    y = adv.copy()
    _kernels.fwht_rows(y, 64)
    g["fwht_adv_out_64"] = y

    # --- quantize_rows / dequantize_rows (_ref.py:57-95) on several input families
    fams = {}
    fams["gauss_bf16"] = bf16_exact(rng.standard_normal((512, 128)) * rng.uniform(0.01, 300, size=(512, 1)))
    ko, vo, _ = generate_kv(default_outlier_spec(), seed=3)
    fams["outlier"] = ko.reshape(-1, 128)[:256]
    kc, vc, _ = generate_kv(default_correlated_spec(), seed=4)
    fams["correlated"] = bf16_exact(kc.reshape(-1, 128)[:256])
    adv = rng.standard_normal((64, 128)) * rng.uniform(0.01, 300, size=(64, 1))
    adv[5] = -3.25                       # constant row (test_kernels.py:39-54)
    adv[9, 17] = 4000.0                  # hard outlier
    adv[10] = np.arange(128) % 16        # grid ties
    adv[11] = np.abs(adv[11]) + 1.0      # all positive -> z clips at 0
    adv[12] = -np.abs(adv[12]) - 1.0     # all negative -> z clips at 15
    adv[13] = 0.0                        # all-zero sentinel
    adv[14] = np.linspace(-7.5, 7.5, 128)  # ties at half steps
    adv[15, :] = 1e-30
    adv[15, 0] = 2e-30                   # f32 scale underflow -> sentinel
    adv[16] = rng.standard_normal(128) * 1e30
    adv[17] = [1.0, 1.0, 1.0, 100.0] * 32  # frozen example generalised (test_int4.py:20-27)
    fams["adversarial"] = adv
    for name, rows in fams.items():
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        p, s, z = _kernels.quantize_rows(rows)
        g[f"q_{name}_in"] = rows
        g[f"q_{name}_packed"] = p
        g[f"q_{name}_scale"] = s
        g[f"q_{name}_zp"] = z
        g[f"q_{name}_deq"] = _kernels.dequantize_rows(p, s, z, rows.shape[1])

    # --- make_signs (rotation.py:81-101): Philox streams pinned as data
    for seed, layer, d, order in ((0, 0, 128, 128), (7, 3, 128, 32), (11, 5, 128, 64), (0, 79, 128, 128), (5, 0, 32, 16)):
        g[f"signs_{seed}_{layer}_{d}_{order}"] = make_signs(seed, layer, d, order)

    # --- apply_block_rotation / inverse (rotation.py:118-159)
    lay = HeadLayout(num_q_heads=32, num_kv_heads=8, head_dim=128, rot_order=128)
    spec = RotationSpec(order=128, signs=make_signs(0, 0, 128, 128))
    xr = bf16_exact(rng.standard_normal((64, 128)))
    g["rot_in"] = xr
    g["rot_fwd"] = apply_block_rotation(xr, lay, spec)
    g["rot_inv"] = apply_inverse_rotation(xr, lay, spec)

    # --- page tables: fused append dumps (cache.py:235-270, 366-399)
    def table_case(tag, layout, tokens, spec, num_pages, seed, seqs=(0,)):
        r = np.random.default_rng(seed)
        t = PageTable(layout, precision=INT4, num_pages=num_pages)
        kv = {}
        for s in seqs:
            t.create_sequence(s)
            k = bf16_exact(r.standard_normal((tokens, layout.num_kv_heads, layout.head_dim)) * 3)
            v = bf16_exact(r.standard_normal((tokens, layout.num_kv_heads, layout.head_dim)))
            kv[s] = (k, v)
            for i in range(tokens):
                t.append_token(s, k[i], v[i], spec=spec)
        path = os.path.join(HERE, f"{tag}.kvpg")
        t.dump(path)
        for s in seqs:
            g[f"tab_{tag}_k_{s}"], g[f"tab_{tag}_v_{s}"] = kv[s]
        return t, kv

    small = HeadLayout(num_q_heads=4, num_kv_heads=2, head_dim=32, rot_order=16, page_tokens=4)
    sspec = RotationSpec(order=16, signs=make_signs(11, 3, 32, 16))
    t_small, kv_small = table_case("small_kv", small, 19, sspec, 8, 1)
    big = HeadLayout(num_q_heads=32, num_kv_heads=8, head_dim=128, rot_order=128, page_tokens=16)
    bspec = RotationSpec(order=128, signs=make_signs(0, 0, 128, 128))
    t_big, kv_big = table_case("big_kv", big, 40, bspec, 4, 2)
    kspec = RotationSpec(order=128, signs=make_signs(0, 1, 128, 128), targets=Targets.KEYS_ONLY)
    t_ko, kv_ko = table_case("big_konly", big, 40, kspec, 4, 3)
    t_plain, kv_plain = table_case("big_plain", big, 40, None, 4, 4)
    h64 = HeadLayout(num_q_heads=4, num_kv_heads=1, head_dim=128, rot_order=64, page_tokens=16)
    s64 = RotationSpec(order=64, signs=make_signs(0, 0, 128, 64))
    t_o64, kv_o64 = table_case("o64_kv", h64, 37, s64, 3, 5)

    # --- decode_step (attention.py:50-87) on those tables
    for tag, table, spec, layout in (("small_kv", t_small, sspec, small), ("big_kv", t_big, bspec, big),
                                     ("big_konly", t_ko, kspec, big), ("big_plain", t_plain, None, big),
                                     ("o64_kv", t_o64, s64, h64)):
        q = bf16_exact(rng.standard_normal((layout.num_q_heads, layout.head_dim)))
        g[f"dec_{tag}_q"] = q
        g[f"dec_{tag}_out"] = decode_step(DecodeRequest(q=q, seq=0), table, spec=spec)
        kf, vf = table.read_sequence(0)
        g[f"dec_{tag}_kread_sum"] = np.array([kf.sum(), vf.sum(), np.abs(kf).sum(), np.abs(vf).sum()])
        g[f"dec_{tag}_fp"] = decode_step_fp(q, kf, vf, layout)

    np.savez_compressed(os.path.join(HERE, "golden_v1.npz"), **g)
    print("kvrot", kvrot.__version__, "numpy", np.__version__, "->", len(g), "arrays")


if __name__ == "__main__":
    sys.exit(main())
