import os, sys
import numpy as np, torch
sys.path.insert(0, "/root/repo" if os.path.exists("/root/repo") else ".")
from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs
from paper_2604_19157_b200.attention import decode_batch
from paper_2604_19157_b200.errors import NonFiniteInputError
MODE = sys.argv[1]  # graph | eager | nonan
N = 4100
B, H, G, D = 3, 8, 4, 128
dev = torch.device("cuda")
layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=D, rot_order=128, page_tokens=16)
spec = RotationSpec(order=128, signs=make_signs(1, 0, D, 128))
t = PageTable(layout, num_pages=(B * (2000 + 20000)) // 16 + 16, device=dev)
torch.manual_seed(0)
for s in range(B):
    t.create_sequence(s)
    L0 = 500 + 700 * s
    t.append_batch([s] * L0, torch.randn(L0, H, D, device=dev).bfloat16(), torch.randn(L0, H, D, device=dev).bfloat16(), spec=spec, check=False)
plan = DecodePlan(t, list(range(B)), extra_tokens=20032, num_splits=int(os.environ.get("SPL", "0")))
print("splits", plan.splits, "max_len", plan.max_len)
qh = torch.empty(B, H * G, D, dtype=torch.bfloat16).pin_memory()
kh = torch.empty(B, H, D, dtype=torch.bfloat16).pin_memory()
vh = torch.empty(B, H, D, dtype=torch.bfloat16).pin_memory()
oh = torch.empty(B, H * G, D).pin_memory()
first_bad = None
for i in range(N):
    qh.copy_(torch.randn(B, H * G, D).bfloat16()); kh.copy_(torch.randn(B, H, D).bfloat16()); vh.copy_(torch.randn(B, H, D).bfloat16())
    if MODE != "nonan" and i % 997 == 13:
        kh[1, 3, 7] = float("nan")
        try:
            plan.step(qh, kh, vh, spec, out=oh, graph=(MODE != "eager")); raise AssertionError("accepted")
        except NonFiniteInputError:
            pass
        continue
    plan.step(qh, kh, vh, spec, out=oh, graph=(MODE != "eager"))
    if i >= 480 or i % 100 == 99:
        torch.cuda.synchronize()
        ref = decode_batch(qh.cuda().float(), t, list(range(B)), spec=spec).cpu()
        err = (oh - ref).abs().amax(dim=2) / ref.abs().amax()
        if float(err.max()) > 1e-5:
            lens = [t.sequence_length(s) for s in range(B)]
            bad = (err > 1e-5).nonzero().tolist()
            print("BAD at step", i, "lens", lens, "rows (seq, qhead)", bad[:12], "max", float(err.max()))
            first_bad = i
            break
print(MODE, "first bad", first_bad, "lens", [t.sequence_length(s) for s in range(B)])
