"""C1 quantize-store timing (4096 tokens x 8 heads, bf16, order 128): rotated and plain,
8 rotating input sets, CUDA-graph replay.  Used under ncu as well (--ncu: few launches)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import HeadLayout, PageTable, RotationSpec, make_signs  # noqa: E402

H, D, P, N = 8, 128, 16, int(os.environ.get("C1_TOKENS", "4096"))
dev = torch.device("cuda")
layout = HeadLayout(num_q_heads=32, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=P)
spec = RotationSpec(order=128, signs=make_signs(0, 0, D, 128))
sets = []
for r in range(8):
    t = PageTable(layout, num_pages=N // P, device=dev)
    t.create_sequence(0)
    t.alloc.plan([0] * N)
    sets.append((t, torch.randn(N, H, D, device=dev).bfloat16(), torch.randn(N, H, D, device=dev).bfloat16(),
                 torch.arange(N, dtype=torch.int64, device=dev)))
ncu = "--ncu" in sys.argv


def run(i, sp):
    t, k, v, sl = sets[i % 8]
    t.store_slots(k, v, sl, sp)


for name, sp in (("rot", spec), ("plain", None)):
    if ncu:
        for i in range(4):
            run(i, sp)
        torch.cuda.synchronize()
        continue
    for i in range(8):
        run(i, sp)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for i in range(64):
            run(i, sp)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 256 * 1e3
    byts = N * (2 * H * D * 2 + H * (D + 10) + 8)
    print(f"{name}: {us:.2f} us  {byts / us / 1e3:.0f} GB/s")
