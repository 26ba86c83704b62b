"""Host-side phases of DecodePlan.step (C2 shapes), GPU drained before each call."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs  # noqa: E402

H, G, D, L = 8, 4, 128, 4096
dev = torch.device("cuda")
layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=16)
spec = RotationSpec(order=128, signs=make_signs(0, 0, D, 128))
t = PageTable(layout, num_pages=(L + 20000) // 16 + 2, device=dev)
t.create_sequence(0)
sl = torch.from_numpy(t.alloc.reserve(0, L)).to(dev)
t.store_slots(torch.randn(L, H, D, device=dev).bfloat16(), torch.randn(L, H, D, device=dev).bfloat16(), sl, spec)
kh = torch.randn(1, H, D).bfloat16().pin_memory()
vh = torch.randn(1, H, D).bfloat16().pin_memory()
qh = torch.randn(1, H * G, D).bfloat16().pin_memory()
oh = torch.empty(1, H * G, D).pin_memory()
plan = DecodePlan(t, [0], extra_tokens=16000)
for _ in range(5):
    plan.step(qh, kh, vh, spec, out=oh, graph=True)
torch.cuda.synchronize()

acc = {}


def tick(name, t0):
    t1 = time.perf_counter_ns()
    acc.setdefault(name, []).append(t1 - t0)
    return t1


ev = torch.cuda.Event()
for i in range(300):
    torch.cuda.synchronize()
    t0 = time.perf_counter_ns()
    slots, fresh = t.alloc.plan(plan.seqs)
    t0 = tick("alloc.plan", t0)
    lens = np.fromiter((t._seq_len[s] for s in plan.seqs), dtype=np.int32, count=1)
    t0 = tick("lens fromiter", t0)
    host_in = [x for x in (qh, kh, vh) if not x.is_cuda]
    lay = plan._step_layout(host_in)
    t0 = tick("layout lookup", t0)
    buf, buf_np, buf_ptr, e, hv = lay["ring"][0]
    e.synchronize()
    t0 = tick("event sync", t0)
    buf_np[:8] = slots.view(np.uint8)
    buf_np[8:12] = lens.view(np.uint8)
    t0 = tick("meta to staging", t0)
    for x, off, n in zip(host_in, lay["offs"], lay["sizes"]):
        x = x if x.is_contiguous() else x.contiguous()
        ctypes.memmove(buf_ptr + off, x.data_ptr(), n)
    t0 = tick("3 memmoves", t0)
    oh.is_pinned()
    t0 = tick("out.is_pinned()", t0)
    torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())
    t0 = tick("raw stream lookup", t0)
    ev.record()
    t0 = tick("Event.record()", t0)
for k, v in acc.items():
    v = sorted(v[50:])
    print(f"{k:22s} median {v[len(v) // 2] / 1e3:6.2f} us")
