"""A long run of the serving step through the native step ring (pinned host q / k / v / out,
page boundaries on the general path, NaN steps rejected), checked against a fresh decode of the
same table state: catches ordering races between consecutive steps that short tests miss."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("mode", ["1", "2"])
def test_step_ring_soak(mode):
    env = dict(os.environ, KVR_STEP_DIRECT=mode, SOAK_EVERY="25")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "soak_step.py"), "3000"], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "soak: 3000 steps" in r.stdout


@pytest.mark.parametrize("device_inputs", [False, True])
def test_serving_soak_with_prefill(device_inputs):
    """Decode steps interleaved on one stream with bulk prefill writes of another sequence and its
    decodes (the pool-write notes gating pre-wait reads), checked against fresh decodes."""
    args = [sys.executable, os.path.join(ROOT, "tools", "soak_serving.py"), "1000"] + (["--device"] if device_inputs
                                                                                        else [])
    r = subprocess.run(args, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "serving soak" in r.stdout and "1000 steps" in r.stdout


def test_learned_step_soak():
    """Row f3 through DecodePlan.step(graph=True): the learned step's graphs must take the staged
    lengths (a graph captured around a host-side length refresh replayed stale lengths)."""
    env = dict(os.environ, SOAK_LEARNED="1", SOAK_EVERY="25")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "soak_step.py"), "1000"], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "soak: 1000 steps" in r.stdout


def test_k1_randomised_stress():
    """Random token counts across both K1 kernels' dispatch range, slot permutations, head counts,
    orders, targets and row families: the fast write equals the exact path (codes / zp bit-exact,
    scales within 2 ulp)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stress_k1.py"), "16"], capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "stress_k1: 16 cases" in r.stdout


def test_decode_randomised_stress():
    """Random ragged batches, head counts, GQA groups, page sizes, orders, targets and split counts:
    the INT4 decode against the flat f64 decode of the same pages, within 1e-5 of max|ref|."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stress_decode.py"), "20"], capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "stress_decode: 20 cases" in r.stdout
