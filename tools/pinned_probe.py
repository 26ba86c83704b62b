"""How fast a kernel reads a small pinned host buffer on this box: the step ring's stage-copy
kernel alone (back to back), and the same with a bandwidth-heavy kernel running beside it."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19157_b200 import _lib  # noqa: E402

dev = torch.device("cuda")
lib = _lib.lib()
for nbytes in (4096, 12288, 65536):
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(10):
        lib.kvr_step_stage  # noqa: B018
    n = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    from paper_2604_19157_b200 import _kernels as K
    f = K._cudart()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        dst.copy_(src, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    t_dma = e0.elapsed_time(e1) / n * 1e3
    print(f"{nbytes} B: cudaMemcpyAsync H2D back to back {t_dma:.2f} us")
