"""Per-CTA timeline of one C2 decode step (globaltimer stamps) -> gpurun_out/trace.txt."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs, _lib  # noqa: E402

H, G, D, L = 8, 4, 128, int(sys.argv[1]) if len(sys.argv) > 1 else 32768
dev = torch.device("cuda")
layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=16)
spec = RotationSpec(order=128, signs=make_signs(0, 0, D, 128))
t = PageTable(layout, num_pages=(L + 15) // 16 + 2, device=dev)
t.create_sequence(0)
for c0 in range(0, L, 8192):
    n = min(8192, L - c0)
    t.append_batch([0] * n, torch.randn(n, H, D, device=dev).bfloat16(), torch.randn(n, H, D, device=dev).bfloat16(),
                   spec=spec, check=False)
plan = DecodePlan(t, [0])
q = torch.randn(1, H * G, D, device=dev).bfloat16()
tr = torch.zeros(plan.splits * H * 8, dtype=torch.int64, device=dev)
for _ in range(3):
    plan.run(q, spec)
torch.cuda.synchronize()
_lib.lib().kvr_debug_decode_trace(ctypes.c_void_p(tr.data_ptr()))
plan.run(q, spec)
torch.cuda.synchronize()
_lib.lib().kvr_debug_decode_trace(None)
a = tr.view(plan.splits * H, 8).cpu().numpy().astype(np.float64)
t0 = a[:, 0].min()
a = (a - t0) / 1000.0
a[a < 0] = np.nan  # unstamped slots
names = ["start", "loop start", "loop end", "partial written", "counter back", "merge done", "end"]
out = [f"splits {plan.splits} ctas {a.shape[0]}"]
for c, nm in enumerate(names):
    col = a[:, c]
    col = col[np.isfinite(col)]
    if col.size:
        out.append(f"{nm:16s}: n {col.size:4d} min {col.min():6.2f} med {np.median(col):6.2f} max {col.max():6.2f} us")
last = np.isfinite(a[:, 5])
if last.any():
    out.append("last CTAs: " + "; ".join(
        " ".join(f"{a[k, c]:.2f}" for c in range(7)) for k in np.nonzero(last)[0][:8]))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    plan.run(q, spec)
e1.record()
torch.cuda.synchronize()
out.append(f"event time per launch (L2-warm): {e0.elapsed_time(e1) / 20 * 1000:.2f} us")
os.makedirs("gpurun_out", exist_ok=True)
open("gpurun_out/trace.txt", "w").write("\n".join(out) + "\n")
print("\n".join(out))
