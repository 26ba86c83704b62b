"""Per-CTA timeline of C2 decode launches (globaltimer/clock64 stamps) -> gpurun_out/trace.txt.

    python tools/trace_decode.py [ctx] [splits ...] [--step] [--steady]

Four independent tables (> 126 MB L2 in total) rotate so the traced launch reads
its KV from HBM, like the bench.  Default: the traced launch starts on an idle
GPU.  --steady: back-to-back launches, the last one traced,
so its start overlaps the previous launch's tail as in the bench's graph replay
(traced inside a CUDA graph of 16 steps; the last one's rows are kept)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs, _lib  # noqa: E402

H, G, D = int(os.environ.get("TR_H", "8")), int(os.environ.get("TR_G", "4")), 128
L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
STEP = "--step" in sys.argv  # fused append + decode (kvr_decode_step)
STEADY = "--steady" in sys.argv
split_list = [int(x) for x in sys.argv[2:] if not x.startswith("--")] or [0]
dev = torch.device("cuda")
layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=16)
spec = RotationSpec(order=128, signs=make_signs(0, 0, D, 128))
tables = []
for _ in range(4):
    t = PageTable(layout, num_pages=(L + 15) // 16 + 2, device=dev)
    t.create_sequence(0)
    for c0 in range(0, L, 8192):
        n = min(8192, L - c0)
        t.append_batch([0] * n, torch.randn(n, H, D, device=dev).bfloat16(),
                       torch.randn(n, H, D, device=dev).bfloat16(), spec=spec, check=False)
    tables.append(t)
q = torch.randn(1, H * G, D, device=dev).bfloat16()
kn = torch.randn(1, H, D, device=dev).bfloat16()
vn = torch.randn(1, H, D, device=dev).bfloat16()
slots = []
if STEP:
    for t in tables:
        sl, fresh = t.alloc.plan([0])
        t._zero_pages(fresh)
        slots.append(torch.from_numpy(sl).to(dev))


def run(plan, k):
    if STEP:
        plan.run_step(q, kn, vn, slots[k], spec)
    else:
        plan.run(q, spec)


out_lines = []
names = {11: "past wait", 14: "wr rows landed", 15: "wr rotated", 8: "wr append done", 13: "q landed", 12: "q prep done", 2: "loop start", 3: "loop end", 4: "M published", 5: "warp partials", 6: "partial stored / split weights", 7: "merge in",
         10: "exit / merged in smem", 9: "merged"}
MHZ = float(os.environ.get("SM_MHZ", "1965"))
lib = _lib.lib()
for splits in split_list:
    plans = [DecodePlan(t, [0], num_splits=splits) for t in tables]
    S = plans[0].splits
    nd = S * H
    tr = torch.zeros((nd + H * G) * 16, dtype=torch.int64, device=dev)
    for k, p in enumerate(plans):
        run(p, k)
    torch.cuda.synchronize()
    if STEADY:  # a CUDA graph of 16 back-to-back steps, traced: the last step's rows survive
        lib.kvr_debug_decode_trace(ctypes.c_void_p(tr.data_ptr()))
        gt = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            with torch.cuda.graph(gt, stream=st):
                for k in range(16):
                    run(plans[k % 4], k % 4)
        torch.cuda.current_stream().wait_stream(st)
        torch.cuda.synchronize()
        gt.replay()
    else:
        for k in range(3):
            run(plans[k], k)
        lib.kvr_debug_decode_trace(ctypes.c_void_p(tr.data_ptr()))
        run(plans[3], 3)
    torch.cuda.synchronize()
    lib.kvr_debug_decode_trace(None)
    raw_all = tr.view(-1, 16).cpu().numpy().astype(np.float64)
    raw = raw_all[:nd]
    t0 = raw[:, 0].min()
    g0 = raw[:, 0] - t0
    out_lines.append(f"== ctx {L} splits {S} ctas {nd} {'fused step' if STEP else 'decode'} "
                     f"({'steady: back-to-back launches' if STEADY else 'launch on an idle GPU'}; HBM-cold KV; "
                     f"clock64 at {MHZ:.0f} MHz; us from the first CTA's entry)")
    out_lines.append(f"{'start':16s}: min {g0.min() / 1e3:6.2f} med {np.median(g0) / 1e3:6.2f} max {g0.max() / 1e3:6.2f} us")
    for k, nm in names.items():
        # rows whose stamp belongs to this launch (the last CTA of an older step can
        # stamp a row after the next step's CTA re-armed it)
        ok = (raw[:, k] > raw[:, 1]) & (raw[:, k] - raw[:, 1] < 1e6)
        if ok.any():
            t = (g0[ok] + (raw[ok, k] - raw[ok, 1]) * 1e3 / MHZ) / 1e3
            out_lines.append(f"{nm:16s}: n {ok.sum():4d} min {t.min():6.2f} med {np.median(t):6.2f} max {t.max():6.2f} us")
    if os.environ.get("TR_BY_SPLIT"):  # rows are cta_id = (b * S + split) * H + h
        rs = raw.reshape(-1, S, H, 16)[0]
        st = (rs[:, :, 0] - t0) / 1e3
        le = st + (rs[:, :, 3] - rs[:, :, 1]) * 1e3 / MHZ / 1e3
        pw = st + (rs[:, :, 11] - rs[:, :, 1]) * 1e3 / MHZ / 1e3
        out_lines.append("  by split: start / past wait / loop end (us, mean over heads)")
        for sp in range(S):
            out_lines.append(f"   split {sp:2d}: {st[sp].mean():6.2f} {pw[sp].mean():6.2f} {le[sp].mean():6.2f}")
    if os.environ.get("TR_MERGE_ROWS"):  # per merger CTA: stamps (ns) relative to 'merge in' (7)
        for r_ in raw[(raw[:, 7] > raw[:, 1])][:6]:
            rel = {k: round((r_[k] - r_[7]) * 1e3 / MHZ, 0) for k in (5, 6, 9) if r_[k] > r_[1]}
            out_lines.append(f"  merger row: {rel}")
    mg = raw_all[nd:]
    mg = mg[mg[:, 0] > 0]
    for k, nm in ((0, "merge entry"), (1, "merge past wait"), (3, "merge lse in"), (2, "merge exit")):
        if len(mg):
            t = (mg[:, k] - t0) / 1e3
            out_lines.append(f"{nm:16s}: n {len(mg):4d} min {t.min():6.2f} med {np.median(t):6.2f} max {t.max():6.2f} us")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for k in range(64):
                run(plans[k % 4], k % 4)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(4):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    out_lines.append(f"graph time per launch (HBM, back to back): {e0.elapsed_time(e1) / 256 * 1000:.2f} us")
os.makedirs("gpurun_out", exist_ok=True)
open("gpurun_out/trace.txt", "a").write("\n".join(out_lines) + "\n")
print("\n".join(out_lines))
