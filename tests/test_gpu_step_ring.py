"""DecodePlan.step's native fast path (kvr_step_ring) vs the general path.

Repeated graph steps with the same pinned host tensors go through one native call per
step (stage + NaN/Inf scan + the fused decode-step launch; modes: 0 graph replay with a
stage-in copy, 1 inputs read in place from pinned memory, 2 a chained stage-copy
kernel).  Every mode must give the bytes of the general path step after step -- outputs,
page contents, lengths -- including across page boundaries (which take the general
path), and a NaN/Inf input must be rejected with nothing committed."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from test_gpu_decode import _build  # noqa: E402
from paper_2604_19157_b200 import errors as E  # noqa: E402
from paper_2604_19157_b200.attention import DecodePlan  # noqa: E402
from paper_2604_19157_b200.rotation import Targets  # noqa: E402


def _run(mode, steps, lens, H=8, G=4, d=128, nan_at=None):
    t, spec, _ = _build(len(lens), lens, H, G, d, 128, 16, "gaussian", Targets.KEYS_AND_VALUES, True, seed=21,
                        extra_pages=len(lens) * (steps // 16 + 2))
    B = len(lens)
    plan = DecodePlan(t, list(range(B)), extra_tokens=steps + 1)
    if mode is None:
        plan.fast_direct = 0
        plan._fast = None
    else:
        plan.fast_direct = mode
    rng = np.random.default_rng(5)
    q = torch.empty((B, G * H, d), dtype=torch.bfloat16).pin_memory()
    k = torch.empty((B, H, d), dtype=torch.bfloat16).pin_memory()
    v = torch.empty((B, H, d), dtype=torch.bfloat16).pin_memory()
    out = torch.empty((B, G * H, d), dtype=torch.float32).pin_memory()
    outs, fast_steps = [], 0
    for i in range(steps):
        q.copy_(torch.tensor(rng.standard_normal(q.shape), dtype=torch.bfloat16))
        k.copy_(torch.tensor(rng.standard_normal(k.shape), dtype=torch.bfloat16))
        v.copy_(torch.tensor(rng.standard_normal(v.shape), dtype=torch.bfloat16))
        if nan_at is not None and i == nan_at:
            k[0, 1, 7] = float("nan")
            before = [t.sequence_length(s) for s in range(B)]
            with pytest.raises(E.NonFiniteInputError):
                plan.step(q, k, v, spec, out=out, graph=True)
            assert [t.sequence_length(s) for s in range(B)] == before
            k[0, 1, 7] = 0.0
        fast_steps += plan._fast is not None and mode is not None
        plan.step(q, k, v, spec, out=out, graph=True)
        torch.cuda.synchronize()
        outs.append(out.clone())
        if mode is None:
            plan._drop_fast()
    pages = t.page_records(range(t.num_pages))
    return torch.stack(outs), pages, [t.sequence_length(s) for s in range(B)], fast_steps


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_step_ring_matches_general_path(mode):
    steps, lens = 40, [45, 130]
    ref_out, ref_pages, ref_lens, _ = _run(None, steps, lens)
    out, pages, ln, fast = _run(mode, steps, lens)
    assert fast >= steps // 2, f"the fast path ran {fast} of {steps} steps"
    assert ln == ref_lens == [L + steps for L in lens]
    assert np.array_equal(pages, ref_pages)
    assert torch.equal(out, ref_out)


@pytest.mark.parametrize("mode", [0, 2])
def test_step_ring_rejects_nonfinite_before_commit(mode):
    steps, lens = 24, [20]
    ref_out, ref_pages, _, _ = _run(None, steps, lens, nan_at=13)
    out, pages, ln, _ = _run(mode, steps, lens, nan_at=13)
    assert ln == [20 + steps]
    assert np.array_equal(pages, ref_pages)
    assert torch.equal(out, ref_out)
