"""Benchmark of the Hadamard-INT4 KV serving hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline workload = BASELINE.json configs[1] (C2): one decode step of a
Llama-3-8B-shaped sequence -- batch 1, 32k cached tokens, GQA 32 q / 8 kv heads,
head_dim 128, Hadamard order 128, page 16, keys AND values rotated.  A step
writes the new token's K/V (fused rotate -> INT4 -> paged store, K1) and runs
the split-K paged INT4 decode with rotated query and inverse-rotated output
(K2+K3).  Metric: algorithmic HBM bytes of the step / step time (GB/s).

* value       device time, inputs resident in HBM, 8 rotating buffer sets
              (> 2x the 126 MB L2) so no step reads L2-warm KV; the K steps
              are replayed from a CUDA graph; max over ranks.
* e2e         the same step through the public API (PageTable.append_batch +
              DecodePlan) with the new token's K/V and q copied from pinned
              host memory and the output copied back, every step.
* roofline    for the dominant kernel (K2 decode) from CUDA events around
              back-to-back launches; traffic from the committed ncu capture.
* cpu_baseline the numpy oracle (port of the reference) on the host.
Multi-GPU (torchrun): every rank serves its own sequence (weak scaling, no
collective on the data path); NCCL only for the barrier / max-time and a
post-timing all_gather of outputs for verification.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H, G, D, ORDER, P = 8, 4, 128, 128, 16
CTX = 32768
NQ = H * G
TOK_BYTES = H * (D + 10)                       # INT4 K+V + sidecar per token (1,104 B)
WRITE_BYTES_PER_TOKEN = 2 * H * D * 2 + TOK_BYTES + 8   # bf16 in + INT4 out + slot id
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def decode_bytes(L: int, batch: int = 1) -> int:
    """Algorithmic bytes of one decode launch."""
    return batch * (L * TOK_BYTES + math.ceil(L / P) * 4 + NQ * D * 2 + NQ * D * 4)


def step_bytes(L: int) -> int:
    return decode_bytes(L) + WRITE_BYTES_PER_TOKEN


def hbm_peak():
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ ours ----

def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs
    from paper_2604_19157_b200.shard import gather_rows, max_over_ranks

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    layout = HeadLayout(num_q_heads=NQ, num_kv_heads=H, head_dim=D, rot_order=ORDER, page_tokens=P)
    spec = RotationSpec(order=ORDER, signs=make_signs(0, 0, D, ORDER))
    L = args.ctx
    R = args.sets
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)

    # ---- R independent buffer sets: a 32k-token sequence + the new token + q
    sets = []
    chunk = 8192
    for r in range(R):
        # headroom for the e2e steps (which append real tokens through the API)
        t = PageTable(layout, num_pages=(L + 1 + P - 1) // P + 64, device=dev)
        t.create_sequence(0)
        for c0 in range(0, L, chunk):
            n = min(chunk, L - c0)
            k = torch.randn((n, H, D), generator=gen, device=dev).to(torch.bfloat16)
            v = torch.randn((n, H, D), generator=gen, device=dev).to(torch.bfloat16)
            t.append_batch([0] * n, k, v, spec=spec, check=False)
        slot_np, fresh = t.alloc.plan([0])          # the step's token: position L
        t._zero_pages(fresh)
        st = dict(table=t, slot=torch.from_numpy(slot_np).to(dev),
                  k=torch.randn((1, H, D), generator=gen, device=dev).to(torch.bfloat16),
                  v=torch.randn((1, H, D), generator=gen, device=dev).to(torch.bfloat16),
                  q=torch.randn((1, NQ, D), generator=gen, device=dev).to(torch.bfloat16),
                  out=torch.empty((1, NQ, D), dtype=torch.float32, device=dev))
        st["plan"] = DecodePlan(t, [0])
        sets.append(st)
    torch.cuda.synchronize()
    t.check_flags()

    def k1(s, sp=spec):
        s["table"].store_slots(s["k"], s["v"], s["slot"], sp)

    def k2(s, sp=spec):
        s["plan"].run(s["q"], sp, out=s["out"])

    def fused(s, sp=spec):
        s["plan"].run_step(s["q"], s["k"], s["v"], s["slot"], sp, out=s["out"])

    def step(i):
        fused(sets[i % R])

    def graph_of(fn, n):
        g = torch.cuda.CUDAGraph()
        stream = torch.cuda.Stream()
        stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(stream):
            for i in range(2):  # warm the launch paths on this stream before capture
                fn(i)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=stream):
                for i in range(n):
                    fn(i)
        torch.cuda.current_stream().wait_stream(stream)
        torch.cuda.synchronize()
        return g

    def timed(fn, count, chunk_steps=256):
        """Device time of `count` calls of fn (replayed from CUDA graphs), max over ranks."""
        n_full, rem = divmod(count, chunk_steps)
        gf = graph_of(fn, chunk_steps) if n_full else None
        gr = graph_of(fn, rem) if rem else None
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n_full):
            gf.replay()
        if gr is not None:
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        return max_over_ranks(e0.elapsed_time(e1), dev)

    # ---- warmup (eager) then the timed K steps
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        ms = timed(step, args.steps)
        # keep the sampler fed while it is running: repeat a short loop for >= 0.5 s
        t0 = time.time()
        extra = 0
        while time.time() - t0 < 0.5 and extra < 50:
            timed(step, 256)
            extra += 1
    ms_per_step = ms / args.steps
    print(f"[bench] step {ms_per_step * 1e3:.2f} us", file=sys.stderr, flush=True)
    Lstep = L + 1
    per_rank_bytes = step_bytes(Lstep)
    value = world * per_rank_bytes / (ms_per_step * 1e-3) / 1e9

    # ---- per-kernel timings (rotated and plain twins)
    n_k = max(args.steps, 512)
    t_fused = ms_per_step
    t_k1 = timed(lambda i: k1(sets[i % R]), n_k) / n_k
    t_k2 = timed(lambda i: k2(sets[i % R]), n_k) / n_k
    t_k1p = timed(lambda i: k1(sets[i % R], None), n_k) / n_k
    t_k2p = timed(lambda i: k2(sets[i % R], None), n_k) / n_k
    t_fp = timed(lambda i: fused(sets[i % R], None), n_k) / n_k
    # restore the rotated token in every set (the plain twin overwrote slot L)
    for s in sets:
        k1(s)
    torch.cuda.synchronize()
    print(f"[bench] k1 {t_k1 * 1e3:.2f} us, k2 {t_k2 * 1e3:.2f} us, k1 plain {t_k1p * 1e3:.2f}, k2 plain "
          f"{t_k2p * 1e3:.2f}, fused {t_fused * 1e3:.2f}, fused plain {t_fp * 1e3:.2f}", file=sys.stderr, flush=True)
    peak, peak_kind = hbm_peak()
    dbytes = step_bytes(Lstep)
    ach = dbytes / (t_fused * 1e-3) / 1e9
    traffic = None
    try:
        with open(NCU_SUMMARY) as f:
            traffic = json.load(f).get("decode_c2_dram_bytes_per_launch")
    except Exception:
        pass

    # ---- e2e through the public API with host buffers
    e2e = e2e_api(torch, layout, spec, dev, sets[0]["table"], args, world)

    # ---- verification gather (after timing; NCCL only here)
    if world > 1:  # every rank's sequence (batch shard) gathered on all ranks
        gathered = gather_rows(sets[0]["out"], [1] * world)
        assert gathered.shape[0] == world
    splits = sets[0]["plan"].splits

    # ---- the other BASELINE configs (parity-test cases, reported in `detail`)
    c1 = c1_quantize_store(torch, layout, spec, dev, gen, timed)
    c3 = c4 = c5 = None
    if not args.quick:
        sets.clear()  # free the headline's buffers first
        torch.cuda.empty_cache()
        c3 = c3_sweep(torch, dev, gen, timed)
        print(f"[bench] C3 {[(r['batch'], r['us'], r['frac']) for r in c3]}", file=sys.stderr, flush=True)
        c5 = c5_long(torch, dev, gen, timed)
        print(f"[bench] C5 {[(r['ctx'], r['rot_order'], r['us'], r['frac']) for r in c5]}", file=sys.stderr, flush=True)
        c4 = c4_llama70b_shard(torch, dev, gen, timed, world)
        print(f"[bench] C4 step {c4['step_us']} us, {c4['tok_per_s_per_gpu']} tok/s/GPU", file=sys.stderr, flush=True)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:  # the CPU baseline: rank 0 at N = 1 only
        cpu = cpu_baseline_c2(args.cpu_seconds)
    if rank != 0:
        return
    clocks = clk.summary()
    line = {
        "metric": "quantize-store + INT4 paged-decode HBM GB/s (one serving decode step, % of HBM roofline)",
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 6),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16 in -> int4 codes (fp32 math, fp16x2 hi/lo tensor-core MMA)",
        "data": "synthetic (torch.randn K/V/q in bf16, seeded per rank)",
        "config": {
            "workload": "BASELINE configs[1] / C2: Llama-3-8B-shaped decode step, batch 1 per GPU, 32768 cached "
                        "tokens (+1 written), GQA 32q/8kv, head_dim 128, Hadamard order 128, page 16, K&V rotated",
            "per_gpu_batch": 1, "ctx": L, "num_q_heads": NQ, "num_kv_heads": H, "head_dim": D,
            "rot_order": ORDER, "page_tokens": P, "decode_splits": splits,
            "l2": f"{R} rotating buffer sets of {step_bytes(Lstep) / 1e6:.1f} MB (> 2x 126 MB L2), CUDA-graph replay",
            "parallelism": f"dp{world} (independent sequences per GPU, no data-path collective)",
            "algorithmic_bytes_per_step": per_rank_bytes,
        },
        "roofline": {"bound": "hbm", "kernel": ("decode_tma_kernel (one kvr_decode_step: fused append + split-K "
                                                "decode + inline split merge by the last CTA)") if splits <= 32 else
                     "decode_tma_kernel + decode_merge_kernel (fused append + split-K decode, then the split merge)",
                     "achieved": round(ach, 1), "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": round(ach / peak, 4), "traffic": traffic, "algorithmic_bytes": dbytes,
                     "avg_launch_us": round(t_fused * 1e3, 3)},
        "cpu_baseline": cpu,
        "e2e": e2e,
        # per step: the fused decode kernel (+ the split-merge kernel above 32 splits;
        # 2..8 merge in a cluster, 9..32 inline in the last CTA)
        "gpu_launches": args.steps * (2 if splits > 32 else 1),
        "clocks": clocks,
        "detail": {
            "k1_write_1tok_us": round(t_k1 * 1e3, 3), "k1_plain_1tok_us": round(t_k1p * 1e3, 3),
            "k2_decode_us": round(t_k2 * 1e3, 3), "k2_plain_us": round(t_k2p * 1e3, 3),
            "k2_overhead_vs_plain": round(t_k2 / t_k2p - 1.0, 4),
            "fused_step_us": round(t_fused * 1e3, 3), "fused_step_plain_us": round(t_fp * 1e3, 3),
            "fused_step_overhead_vs_plain": round(t_fused / t_fp - 1.0, 4),
            "c1_quantize_store": c1,
            "c3_concurrency_sweep": c3,
            "c4_llama70b_8gpu_shard": c4,
            "c5_long_context_1kv_per_gpu": c5,
        },
    }
    print(json.dumps(line), flush=True)


def build_table(torch, layout, spec, dev, gen, B, L, extra_tokens=1, chunk=16384):
    """B sequences of L cached tokens (random bf16 K/V written through K1), with
    page room for `extra_tokens` more per sequence."""
    from paper_2604_19157_b200 import PageTable

    P, Hh, Dd = layout.page_tokens, layout.num_kv_heads, layout.head_dim
    t = PageTable(layout, num_pages=B * -(-(L + extra_tokens) // P), device=dev)
    for b in range(B):
        t.create_sequence(b)
        slots = torch.from_numpy(t.alloc.reserve(b, L)).to(dev)
        for c0 in range(0, L, chunk):
            n = min(chunk, L - c0)
            k = torch.randn((n, Hh, Dd), generator=gen, device=dev).to(torch.bfloat16)
            v = torch.randn((n, Hh, Dd), generator=gen, device=dev).to(torch.bfloat16)
            t.store_slots(k, v, slots[c0:c0 + n], spec)
    return t


def clone_table(torch, t):
    """Same allocator state and page contents in a fresh pool (another layer's cache)."""
    from paper_2604_19157_b200 import PageTable

    c = PageTable(t.layout, num_pages=t.num_pages, device=t.device)
    c.pool.copy_(t.pool)
    c.alloc.seq_pages = {s: list(p) for s, p in t.alloc.seq_pages.items()}
    c.alloc.seq_len = dict(t.alloc.seq_len)
    c.alloc.free = list(t.alloc.free)
    return c


def decode_case(torch, dev, tables, spec, timed, fused=False, n=256, gen=None):
    """Device time of one decode (or fused append + decode) launch per table, with
    the tables replayed round robin (rotated and plain twin); returns a dict."""
    from paper_2604_19157_b200 import DecodePlan

    lay = tables[0].layout
    seqs = sorted(tables[0].alloc.seq_pages)
    B = len(seqs)
    cases = []
    for t in tables:
        c = {"table": t}
        if fused:
            sl, fresh = t.alloc.plan(seqs)
            t._zero_pages(fresh)
            c["slot"] = torch.from_numpy(sl).to(dev)
            c["k"] = torch.randn((B, lay.num_kv_heads, lay.head_dim), generator=gen, device=dev).to(torch.bfloat16)
            c["v"] = torch.randn((B, lay.num_kv_heads, lay.head_dim), generator=gen, device=dev).to(torch.bfloat16)
        c["plan"] = DecodePlan(t, seqs)
        c["q"] = torch.randn((B, lay.num_q_heads, lay.head_dim), generator=gen, device=dev).to(torch.bfloat16)
        c["out"] = torch.empty((B, lay.num_q_heads, lay.head_dim), dtype=torch.float32, device=dev)
        cases.append(c)
    R = len(cases)

    def one(i, sp):
        c = cases[i % R]
        if fused:
            c["plan"].run_step(c["q"], c["k"], c["v"], c["slot"], sp, out=c["out"])
        else:
            c["plan"].run(c["q"], sp, out=c["out"])

    t_rot = timed(lambda i: one(i, spec), n) / n
    t_pl = timed(lambda i: one(i, None), n) / n
    if fused:  # restore the rotated new token the plain twin overwrote
        for i in range(R):
            one(i, spec)
        torch.cuda.synchronize()
    L = max(tables[0].alloc.seq_len.values())
    Hh, G = lay.num_kv_heads, lay.num_q_heads // lay.num_kv_heads
    tokb = Hh * (lay.head_dim + 10)
    byts = B * (L * tokb + -(-L // lay.page_tokens) * 4 + lay.num_q_heads * lay.head_dim * (2 + 4))
    if fused:
        byts += B * (2 * Hh * lay.head_dim * 2 + tokb + 8)
    peak, _ = hbm_peak()
    return {"batch": B, "ctx": L, "num_kv_heads": Hh, "q_per_kv": G, "rot_order": lay.rot_order,
            "splits": cases[0]["plan"].splits, "algorithmic_bytes": byts,
            "us": round(t_rot * 1e3, 3), "plain_us": round(t_pl * 1e3, 3),
            "GBps": round(byts / (t_rot * 1e-3) / 1e9, 1), "frac": round(byts / (t_rot * 1e-3) / 1e9 / peak, 4),
            "overhead_vs_plain": round(t_rot / t_pl - 1.0, 4), "tok_per_s": round(B / (t_rot * 1e-3), 1),
            "l2": f"{R} rotating table(s) of {byts / 1e6:.0f} MB"}


def c3_sweep(torch, dev, gen, timed):
    """BASELINE configs[2]: batch 1/16/64/256 x 8k context decode, Hadamard vs plain INT4."""
    from paper_2604_19157_b200 import HeadLayout, RotationSpec, make_signs

    layout = HeadLayout(num_q_heads=NQ, num_kv_heads=H, head_dim=D, rot_order=ORDER, page_tokens=P)
    spec = RotationSpec(order=ORDER, signs=make_signs(0, 0, D, ORDER))
    out = []
    for B in (1, 16, 64, 256):
        reps = max(1, -(-300_000_000 // (B * 8192 * TOK_BYTES)))  # > 2x L2 across the rotation
        base = build_table(torch, layout, spec, dev, gen, B, 8192)
        tables = [base] + [clone_table(torch, base) for _ in range(reps - 1)]
        out.append(decode_case(torch, dev, tables, spec, timed, gen=gen))
        del tables, base
        torch.cuda.empty_cache()
    return out


def c4_llama70b_shard(torch, dev, gen, timed, world):
    """BASELINE configs[3] at its 8-GPU shard size on this GPU: Llama-3-70B KV geometry
    (8 kv heads, 64 q heads, d 128), 128 sequences / 8 GPUs = 16 sequences x 16k
    context, 80 layers; one step = the fused append + decode of every layer."""
    from paper_2604_19157_b200 import HeadLayout, RotationSpec, make_signs

    layers, B, L = 80, 128 // 8, 16384
    layout = HeadLayout(num_q_heads=64, num_kv_heads=8, head_dim=D, rot_order=ORDER, page_tokens=P)
    spec = RotationSpec(order=ORDER, signs=make_signs(0, 0, D, ORDER))
    base = build_table(torch, layout, spec, dev, gen, B, L)
    tables = [base] + [clone_table(torch, base) for _ in range(layers - 1)]
    r = decode_case(torch, dev, tables, spec, timed, fused=True, n=layers * 4, gen=gen)
    step_us = r["us"] * layers
    res = {"layers": layers, "sequences_per_gpu": B, "ctx": L, "q_heads": 64, "kv_heads": 8,
           "layer_step_us": r["us"], "layer_plain_us": r["plain_us"], "step_us": round(step_us, 1),
           "tok_per_s_per_gpu": round(B / (step_us * 1e-6), 1), "GBps": r["GBps"], "frac": r["frac"],
           "overhead_vs_plain": r["overhead_vs_plain"], "splits": r["splits"],
           "bytes_per_step": r["algorithmic_bytes"] * layers,
           "note": "per-GPU shard of the 8-GPU configuration (128 x 16k x 80 layers = 186 GB does not fit "
                   "one 180 GB GPU); 80 layer caches, each step runs all 80 fused append+decode launches"}
    del tables, base
    torch.cuda.empty_cache()
    return res


def c5_long(torch, dev, gen, timed):
    """BASELINE configs[4]: one request at 128k / 1M tokens, KV heads sharded 8 ways
    (this GPU: 1 kv head + its 4 q heads), split-K decode, Hadamard order 64 / 128."""
    from paper_2604_19157_b200 import HeadLayout, RotationSpec, make_signs

    out = []
    for L in (131072, 1048576):
        for order in (128, 64):
            layout = HeadLayout(num_q_heads=4, num_kv_heads=1, head_dim=D, rot_order=order, page_tokens=P)
            spec = RotationSpec(order=order, signs=make_signs(0, 0, D, order))
            reps = max(2, -(-300_000_000 // (L * (D + 10))))
            base = build_table(torch, layout, spec, dev, gen, 1, L)
            tables = [base] + [clone_table(torch, base) for _ in range(reps - 1)]
            out.append(decode_case(torch, dev, tables, spec, timed, gen=gen, n=128))
            del tables, base
            torch.cuda.empty_cache()
    return out


def c1_quantize_store(torch, layout, spec, dev, gen, timed):
    """configs[0] shape on the GPU: 4096 tokens x 8 kv heads, order 128, bf16 in."""
    from paper_2604_19157_b200 import PageTable

    n_tok, R = 4096, 8
    sets = []
    for r in range(R):
        t = PageTable(layout, num_pages=n_tok // P, device=dev)
        t.create_sequence(0)
        slots = torch.arange(n_tok, dtype=torch.int64, device=dev)
        t.alloc.plan([0] * n_tok)
        k = torch.randn((n_tok, H, D), generator=gen, device=dev).to(torch.bfloat16)
        v = torch.randn((n_tok, H, D), generator=gen, device=dev).to(torch.bfloat16)
        sets.append((t, k, v, slots))
    n = 256
    t_rot = timed(lambda i: sets[i % R][0].store_slots(sets[i % R][1], sets[i % R][2], sets[i % R][3], spec), n) / n
    t_pl = timed(lambda i: sets[i % R][0].store_slots(sets[i % R][1], sets[i % R][2], sets[i % R][3], None), n) / n
    byts = n_tok * WRITE_BYTES_PER_TOKEN
    peak, _ = hbm_peak()
    # K4 flatten-dequant of the same 4096 tokens back to bf16 (stored space)
    import ctypes

    from paper_2604_19157_b200 import _kernels, _lib
    outs = []
    for t, _, _, _ in sets:
        bt, lens, ml = t.block_table([0])
        outs.append((t, bt, lens, ml, torch.empty((1, n_tok, H, D), dtype=torch.bfloat16, device=dev),
                     torch.empty((1, n_tok, H, D), dtype=torch.bfloat16, device=dev)))

    def deq(i):
        t, bt, lens, ml, ko, vo = outs[i % R]
        _lib.check(_lib.lib().kvr_dequantize_pages(ctypes.byref(t.desc), _kernels.ptr(bt), bt.shape[1],
                                                   _kernels.ptr(lens), 1, ml, _kernels.ptr(ko), _kernels.ptr(vo),
                                                   _lib.KVR_BF16, _kernels.stream_ptr()))
    t_dq = timed(deq, n) / n
    dq_bytes = n_tok * (TOK_BYTES + 2 * H * D * 2) + (n_tok // P) * 4
    return {"tokens": n_tok, "algorithmic_bytes": byts, "rot_us": round(t_rot * 1e3, 3),
            "dequant_us": round(t_dq * 1e3, 3), "dequant_GBps": round(dq_bytes / (t_dq * 1e-3) / 1e9, 1),
            "dequant_frac": round(dq_bytes / (t_dq * 1e-3) / 1e9 / peak, 4),
            "plain_us": round(t_pl * 1e3, 3), "rot_GBps": round(byts / (t_rot * 1e-3) / 1e9, 1),
            "plain_GBps": round(byts / (t_pl * 1e-3) / 1e9, 1), "rot_frac": round(byts / (t_rot * 1e-3) / 1e9 / peak, 4),
            "overhead_vs_plain": round(t_rot / t_pl - 1.0, 4)}


def e2e_api(torch, layout, spec, dev, table, args, world):
    """Public-API step with host buffers: H2D of the new K/V and q, DecodePlan.step
    (slot allocation + one fused append+decode launch), D2H of the output."""
    from paper_2604_19157_b200 import DecodePlan

    steps = min(args.steps, 200)
    kh = torch.randn((1, H, D)).to(torch.bfloat16).pin_memory()
    vh = torch.randn((1, H, D)).to(torch.bfloat16).pin_memory()
    qh = torch.randn((1, NQ, D)).to(torch.bfloat16).pin_memory()
    oh = torch.empty((1, NQ, D), dtype=torch.float32).pin_memory()
    free_before = list(table.alloc.free)
    base_len = table.alloc.seq_len[0]
    base_pages = list(table.alloc.seq_pages[0])
    plan = DecodePlan(table, [0], extra_tokens=steps + 8)

    def one():
        # host bookkeeping (slot allocation, page table) per step; q/k/v and the slot /
        # length metadata go to the device in one pinned copy, the fused kernel writes
        # the output straight into the pinned host tensor (both cross the bus every step)
        plan.step(qh, kh, vh, spec, out=oh, graph=True)

    for _ in range(3):
        one()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(steps):
        one()
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    ms = max(e0.elapsed_time(e1), wall) / steps
    # roll the table back
    table.alloc.free = free_before
    table.alloc.seq_len[0] = base_len
    table.alloc.seq_pages[0] = base_pages
    L = base_len + steps
    byts = step_bytes(L)
    return {"value": round(world * byts / (ms * 1e-3) / 1e9, 2), "unit": "GB/s", "ms_per_step": round(ms, 4),
            "h2d_bytes_per_step": kh.numel() * 2 + vh.numel() * 2 + qh.numel() * 2 + 12,  # + slot id, length
            "d2h_bytes_per_step": oh.numel() * 4,
            "api": "DecodePlan.step(graph=True) (fused append + decode) with pinned host buffers",
            "steps": steps}


# ----------------------------------------------------- CPU oracle timing ----

def _cpu_threads():
    try:
        from threadpoolctl import threadpool_info

        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count() or 1


class CpuOracleSequence:
    """A C2-shaped sequence in the numpy oracle's page pool (filled once, untimed)."""

    def __init__(self, L, rng, signs, extra_tokens=64):
        from oracle import kvrot_oracle as O

        self.O, self.rng, self.signs = O, rng, signs
        self.pages = O.OraclePages(NQ, H, D, ORDER, P, (L + extra_tokens + P - 1) // P)
        self.pages.create_sequence(0)
        k = rng.standard_normal((L, H, D))
        v = rng.standard_normal((L, H, D))
        kp, ks, kz = O.quantize_rows(O.rotate_rows(k.reshape(-1, D), ORDER, signs))
        vp, vs, vz = O.quantize_rows(O.rotate_rows(v.reshape(-1, D), ORDER, signs))
        full = L // P
        for pi in range(full):
            sl = slice(pi * P * H, (pi + 1) * P * H)
            pg = self.pages._blank()
            pg["k_payload"][:] = kp[sl].reshape(P, H, D // 2)
            pg["k_scale"][:] = ks[sl].reshape(P, H)
            pg["k_zp"][:] = kz[sl].reshape(P, H)
            pg["v_payload"][:] = vp[sl].reshape(P, H, D // 2)
            pg["v_scale"][:] = vs[sl].reshape(P, H)
            pg["v_zp"][:] = vz[sl].reshape(P, H)
            pid = self.pages.free.pop(0)
            self.pages.pages[pid] = pg
            self.pages.seq_pages[0].append(pid)
        self.pages.seq_len[0] = full * P
        for t in range(full * P, L):
            self.pages.append_token(0, k[t], v[t], signs=signs)

    def step(self):
        """Timed: one token write (rotate + quantize + store) + one decode over the sequence."""
        newk = self.rng.standard_normal((H, D))
        newv = self.rng.standard_normal((H, D))
        q = self.rng.standard_normal((NQ, D))
        t0 = time.perf_counter()
        self.pages.append_token(0, newk, newv, signs=self.signs)
        self.O.decode_step(self.pages, 0, q, signs=self.signs)
        return time.perf_counter() - t0


def _cpu_kernels():
    """Use the reference's compiled kernels (oracle/_ref) when they were built;
    returns the cpu_baseline kind."""
    from oracle import build_ref
    from oracle import kvrot_oracle as O

    mod = build_ref.load()
    if mod is None:
        return "port"
    O.use_reference_kernels(mod)
    return "reference"


_KIND_NOTE = {"reference": "the reference's compiled kernels (oracle/_ref: _core.pyx built from the reference "
                           "sources) for rotate / quantize / dequantize + the numpy restatement of "
                           "attention.decode_step's contraction",
              "port": "the numpy oracle port of the reference"}


def cpu_baseline_c2(seconds: float):
    from oracle import kvrot_oracle as O

    kind = _cpu_kernels()

    rng = np.random.default_rng(0)
    signs = O.make_signs(0, 0, D, ORDER)
    L = CTX
    seq = CpuOracleSequence(L, rng, signs)
    times = []
    t_start = time.perf_counter()
    while not times or (time.perf_counter() - t_start < seconds and len(times) < 40):
        times.append(seq.step())
    t = float(np.median(times))
    return {"value": round(step_bytes(L + 1) / t / 1e9, 4), "unit": "GB/s", "cores": _cpu_threads(),
            "kind": kind, "sample": f"{len(times)} full C2 steps (1-token write + decode over {L + 1} tokens) with "
                                    f"{_KIND_NOTE[kind]} (numpy/OpenBLAS threads), median {t * 1e3:.1f} ms/step"}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm (numpy port in oracle/) on the host cores,
    same metric/config; rank 0 only."""
    if rank != 0:
        return
    from oracle import kvrot_oracle as O

    kind = _cpu_kernels()
    rng = np.random.default_rng(0)
    signs = O.make_signs(0, 0, D, ORDER)
    # bound the run to a few minutes: each step is a full C2 step when affordable,
    # otherwise a step over a shorter context (stated in `sample`)
    budget = 120.0
    probe = CpuOracleSequence(4096, rng, signs).step()
    per_tok = probe / 4096
    L = int(min(CTX, max(1024, budget / max(args.steps + args.warmup, 1) / per_tok)))
    seq = CpuOracleSequence(L, rng, signs, extra_tokens=args.steps + args.warmup + 16)
    for _ in range(args.warmup):
        seq.step()
    ts = [seq.step() for _ in range(args.steps)]
    total = float(np.sum(ts))
    ms = total / args.steps * 1e3
    val = step_bytes(L + 1) / (total / args.steps) / 1e9
    line = {
        "impl": "reference", "metric": "quantize-store + INT4 paged-decode HBM GB/s (one serving decode step, "
                                       "% of HBM roofline)",
        "value": round(val, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 (reference numpy arithmetic)", "data": "synthetic (numpy standard normal)",
        "config": {"workload": "BASELINE configs[1] / C2 decode step on the host CPU (reference algorithm)",
                   "ctx": L, "num_q_heads": NQ, "num_kv_heads": H, "head_dim": D, "rot_order": ORDER,
                   "page_tokens": P},
        "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": _cpu_threads(), "kind": kind,
                         "sample": f"{args.steps} steps, each a 1-token write + decode over {L + 1} tokens, "
                                   f"{_KIND_NOTE[kind]}"
                                   + ("" if L == CTX else f" (context bounded from {CTX} to fit the time budget)")},
        "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ctx", type=int, default=CTX)
    ap.add_argument("--sets", type=int, default=8)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--quick", action="store_true", help="headline + C1 only (skip the C3/C4/C5 detail configs)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
