"""Where the host time of DecodePlan.step goes (C2 shapes, graph=True, pinned host in/out):
wall time per step without a profiler, then a cProfile of the same loop."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs  # noqa: E402

H, G, D, L = 8, 4, 128, int(os.environ.get("CTX", "32768"))
dev = torch.device("cuda")
layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=16)
spec = RotationSpec(order=128, signs=make_signs(0, 0, D, 128))
R = int(os.environ.get("TABLES", "1"))  # the bench rotates 8 tables (> 2x L2)
tables = []
for _ in range(R):
    t = PageTable(layout, num_pages=(L + 8000) // 16 + 2, device=dev)
    t.create_sequence(0)
    sl = torch.from_numpy(t.alloc.reserve(0, L)).to(dev)
    for c0 in range(0, L, 8192):
        t.store_slots(torch.randn(8192, H, D, device=dev).bfloat16(), torch.randn(8192, H, D, device=dev).bfloat16(),
                      sl[c0:c0 + 8192], spec)
    tables.append(t)
DEVIN = os.environ.get("DEVIN", "0") == "1"  # inputs already on the device (no stage-in copy)
kh = torch.randn(1, H, D).bfloat16().pin_memory()
vh = torch.randn(1, H, D).bfloat16().pin_memory()
qh = torch.randn(1, H * G, D).bfloat16().pin_memory()
oh = torch.empty(1, H * G, D).pin_memory()
if DEVIN:
    kh, vh, qh = kh.cuda(), vh.cuda(), qh.cuda()
plans = [DecodePlan(t, [0], extra_tokens=7000) for t in tables]
check = os.environ.get("CHECK", "1") == "1"
for i in range(10 * R):
    plans[i % R].step(qh, kh, vh, spec, out=oh, graph=True, check=check)
torch.cuda.synchronize()
N = 2000
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for i in range(N):
    plans[i % R].step(qh, kh, vh, spec, out=oh, graph=True, check=check)
e1.record()
torch.cuda.synchronize()
print(f"devin={DEVIN} side={os.environ.get('KVR_STEP_SIDE_COPY', '0')} check={check} tables={R}: {(time.perf_counter() - t0) / N * 1e6:.1f} us/step wall, "
      f"{e0.elapsed_time(e1) / N * 1e3:.1f} us/step device (graph=True)")
import numpy as _np
from paper_2604_19157_b200 import _lib as _L
_t = _np.zeros(4)
_L.lib().kvr_debug_step_ring_times(_t.ctypes.data)
print("ring run ns (stage, meta, launch, record):", _t.round(0))
t0 = time.perf_counter()
for i in range(N):
    plans[i % R]._fast_step(plans[i % R]._fast) if plans[i % R]._fast else None
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for i in range(N):
    plans[i % R].step(qh, kh, vh, spec, out=oh, graph=True, check=check)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
