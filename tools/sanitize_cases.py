"""Small launches of every kernel path for compute-sanitizer (memcheck / racecheck / synccheck):
K1 (mma.sync and tcgen05 kernels, rotated and plain), the exact store, K4 dequant, and the
decode in its three split-merge forms (thread-block cluster <= 8 splits, inline last-CTA
merge 9..32, merge kernel > 32) plus the fused step and the step ring."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs, _lib  # noqa: E402

dev = torch.device("cuda")
H, G, D, P = 2, 4, 128, 16
layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=P)
spec = RotationSpec(order=128, signs=make_signs(0, 0, D, 128))
L = int(os.environ.get("SAN_L", "2048"))
t = PageTable(layout, num_pages=L // P + 16, device=dev)
t.create_sequence(0)
k = torch.randn(L, H, D, device=dev).bfloat16()
v = torch.randn(L, H, D, device=dev).bfloat16()
for impl in ((1,) if os.environ.get("SAN_SKIP_TC") else (1, 2)):  # mma.sync K1, tcgen05 K1
    _lib.lib().kvr_debug_set_k1_impl(impl)
    sl = torch.arange(L, dtype=torch.int64, device=dev)
    t.alloc.seq_len[0] = 0
    t.alloc.seq_pages[0] = []
    t.alloc.free = list(range(t.num_pages))
    t.store_slots(k, v, torch.from_numpy(t.alloc.reserve(0, L)).to(dev), spec)
    t.store_slots(k, v, sl, None)
    torch.cuda.synchronize()
_lib.lib().kvr_debug_set_k1_impl(0)
t.alloc.seq_len[0] = 0
t.alloc.seq_pages[0] = []
t.alloc.free = list(range(t.num_pages))
t.store_slots(k, v, torch.from_numpy(t.alloc.reserve(0, L)).to(dev), spec)
t.store_slots(k[:64], v[:64], torch.arange(64, dtype=torch.int64, device=dev), spec, exact=True)
kd, vd = t.read_sequence_device([0], torch.bfloat16)  # K4
q = torch.randn(1, H * G, D, device=dev).bfloat16()
for splits in (1, 4, 12, 48):  # single CTA, cluster, inline merge, merge kernel
    plan = DecodePlan(t, [0], num_splits=splits)
    plan.run(q, spec)
    torch.cuda.synchronize()
# fused step + the native step ring (pinned host inputs, graph steps)
plan = DecodePlan(t, [0], extra_tokens=40)
qh = torch.randn(1, H * G, D).bfloat16().pin_memory()
kh = torch.randn(1, H, D).bfloat16().pin_memory()
vh = torch.randn(1, H, D).bfloat16().pin_memory()
oh = torch.empty(1, H * G, D).pin_memory()
for _ in range(12):
    plan.step(qh, kh, vh, spec, out=oh, graph=True)
torch.cuda.synchronize()
# row f3: the learned-R K1 (tcgen05, T in shared memory; V plain / Hadamard / T) and the fused
# learned decode (T bulk-copied into shared memory; q T in the prologue, the value branch's inverse
# in every merge path: single CTA, cluster, flag-in-data merge, clamped split count)
from paper_2604_19157_b200 import Targets  # noqa: E402

qr_, rr_ = np.linalg.qr(np.random.default_rng(5).standard_normal((D, D)))
R = qr_ * np.sign(np.diag(rr_))
for tg, lv in ((Targets.KEYS_AND_VALUES, False), (Targets.KEYS_AND_VALUES, True), (Targets.KEYS_ONLY, False)):
    lspec = RotationSpec(order=128, signs=spec.signs, learned=R, targets=tg, learned_values=lv)
    t.alloc.seq_len[0] = 0
    t.alloc.seq_pages[0] = []
    t.alloc.free = list(range(t.num_pages))
    t.store_slots(k, v, torch.from_numpy(t.alloc.reserve(0, L)).to(dev), lspec)
    for splits in (1, 4, 12, 48):
        DecodePlan(t, [0], num_splits=splits).run(q, lspec)
    torch.cuda.synchronize()
# BF16 pool: the tuned decode (TMA cells, split-K + merge)
from paper_2604_19157_b200.cache import BF16  # noqa: E402

tb = PageTable(layout, num_pages=L // P + 4, device=dev, precision=BF16)
tb.create_sequence(0)
tb.store_slots(k, v, torch.from_numpy(tb.alloc.reserve(0, L)).to(dev), None)
for splits in (1, 12):
    DecodePlan(tb, [0], num_splits=splits).run(q, None)
torch.cuda.synchronize()
print("sanitize cases done")
