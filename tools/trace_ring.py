"""Per-CTA timeline of the e2e serving step (DecodePlan.step with pinned host q / k / v / out
through the native step ring), C2 shapes: where the ring's extra device time goes.

    KVR_STEP_DIRECT=1|2 python tools/trace_ring.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs, _lib  # noqa: E402

H, G, D, L = 8, 4, 128, 32768
dev = torch.device("cuda")
layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=16)
spec = RotationSpec(order=128, signs=make_signs(0, 0, D, 128))
t = PageTable(layout, num_pages=(L + 4000) // 16 + 2, device=dev)
t.create_sequence(0)
sl = torch.from_numpy(t.alloc.reserve(0, L)).to(dev)
for c0 in range(0, L, 8192):
    t.store_slots(torch.randn(8192, H, D, device=dev).bfloat16(), torch.randn(8192, H, D, device=dev).bfloat16(),
                  sl[c0:c0 + 8192], spec)
kh = torch.randn(1, H, D).bfloat16().pin_memory()
vh = torch.randn(1, H, D).bfloat16().pin_memory()
qh = torch.randn(1, H * G, D).bfloat16().pin_memory()
oh = torch.empty(1, H * G, D).pin_memory()
plan = DecodePlan(t, [0], extra_tokens=3000)
for _ in range(40):
    plan.step(qh, kh, vh, spec, out=oh, graph=True)
torch.cuda.synchronize()
S = plan.splits
nd = S * H
tr = torch.zeros(max((nd + H * G) * 16, 8192 + 16), dtype=torch.int64, device=dev)
lib = _lib.lib()
lib.kvr_debug_decode_trace(ctypes.c_void_p(tr.data_ptr()))
# steady state: 12 back-to-back ring steps (no page boundary inside: the fast path throughout)
while (t.sequence_length(0) + 1) % 16 == 0 or (t.sequence_length(0) + 13) // 16 != (t.sequence_length(0) + 1) // 16:
    plan.step(qh, kh, vh, spec, out=oh, graph=True)
for _ in range(12):
    plan.step(qh, kh, vh, spec, out=oh, graph=True)
torch.cuda.synchronize()
lib.kvr_debug_decode_trace(None)
rall = tr.cpu().numpy().astype(np.float64)
raw = rall[:(nd + H * G) * 16].reshape(-1, 16)[:nd]
cp = rall[8192:8195]
MHZ = 1965.0
t0 = raw[:, 0].min()
g0 = raw[:, 0] - t0
names = {11: "past wait", 14: "wr rows landed", 15: "wr rotated", 8: "wr append done", 13: "q landed",
         12: "q prep done", 2: "loop start", 3: "loop end", 4: "M published", 5: "warp partials", 7: "merge in",
         9: "merged"}
print(f"ring mode {os.environ.get('KVR_STEP_DIRECT', '2')}, splits {S}: us from the first CTA's entry")
print(f"{'start':16s}: min {g0.min() / 1e3:6.2f} med {np.median(g0) / 1e3:6.2f} max {g0.max() / 1e3:6.2f}")
if cp[0] > 0:  # the last step's stage-copy kernel (globaltimer, same clock as 'start')
    print(f"copy kernel     : entry {(cp[0] - t0) / 1e3:6.2f} stores done {(cp[1] - t0) / 1e3:6.2f} past wait {(cp[2] - t0) / 1e3:6.2f}")
for k, nm in names.items():
    ok = (raw[:, k] > raw[:, 1]) & (raw[:, k] - raw[:, 1] < 1e6)
    if ok.any():
        tt = (g0[ok] + (raw[ok, k] - raw[ok, 1]) * 1e3 / MHZ) / 1e3
        print(f"{nm:16s}: n {ok.sum():4d} min {tt.min():6.2f} med {np.median(tt):6.2f} max {tt.max():6.2f}")
