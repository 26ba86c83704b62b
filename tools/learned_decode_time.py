"""Row f3 decode timing at the C2 shape (1 x 32,768 tokens, 8 kv heads, G = 4): the fused
learned decode (kvr_paged_decode_learned) against the unfused route and the Hadamard-only
decode, CUDA-graph replay over 8 rotating tables (> 2x L2).  Prints microseconds per decode."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs  # noqa: E402

H, G, D, P, L = 8, 4, 128, 16, int(os.environ.get("LD_CTX", "32768"))
dev = torch.device("cuda")
layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=P)
qm, rm = np.linalg.qr(np.random.default_rng(7).standard_normal((D, D)))
had = RotationSpec(order=128, signs=make_signs(0, 0, D, 128))
lrn = RotationSpec(order=128, signs=had.signs, learned=qm * np.sign(np.diag(rm)), learned_values=True)
plans = []
for r in range(8):
    t = PageTable(layout, num_pages=L // P + 2, device=dev)
    t.create_sequence(0)
    for c0 in range(0, L, 8192):
        n = min(8192, L - c0)
        t.append_batch([0] * n, torch.randn(n, H, D, device=dev).bfloat16(), torch.randn(n, H, D, device=dev).bfloat16(),
                       spec=had, check=False)
    plans.append(DecodePlan(t, [0]))
q = torch.randn(1, H * G, D, device=dev).bfloat16()


def us(spec, mode):
    os.environ["KVR_LEARNED_DECODE"] = mode
    for p in plans:
        p.run(q, spec)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for i in range(64):
            plans[i % 8].run(q, spec)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 320 * 1e3


print(f"ctx {L}: hadamard {us(had, 'fused'):.2f} us, learned fused {us(lrn, 'fused'):.2f} us, "
      f"learned unfused {us(lrn, 'unfused'):.2f} us")
