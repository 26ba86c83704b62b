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


def headline_config(world: int) -> dict:
    """The workload's config dict, identical for the repo arm and the reference arm."""
    return {
        "workload": "BASELINE configs[1] / C2: Llama-3-8B-shaped decode step, batch 1 per GPU, 32768 cached "
                    "tokens (+1 written), GQA 32q/8kv, head_dim 128, Hadamard order 128, page 16, K&V rotated",
        "per_gpu_batch": 1, "ctx": CTX, "num_q_heads": NQ, "num_kv_heads": H, "head_dim": D,
        "rot_order": ORDER, "page_tokens": P,
        "l2": "inputs rotate over buffer sets larger than 2x the 126 MB L2 (GPU arm)",
        "parallelism": f"dp{world} (independent sequences per GPU, no data-path collective)",
        "algorithmic_bytes_per_step": step_bytes(CTX + 1),
    }


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
    L = CTX
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

    def timed_in_graph(fn, count):
        """Device time of `count` calls of fn inside ONE graph that also holds the timing events
        (recorded as graph nodes) after one untimed step: the graph's own launch is outside the
        window and the first timed step has a predecessor to overlap with, as in steady state."""
        import ctypes as _ct
        from paper_2604_19157_b200 import _kernels as _K
        rt = _K._cudart()
        rt.cudaEventRecordWithFlags.argtypes = [_ct.c_void_p, _ct.c_void_p, _ct.c_uint]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        e1.record()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        stream = torch.cuda.Stream()
        stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(stream):
            for i in range(2):
                fn(i)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=stream):
                fn(count)  # untimed predecessor
                rt.cudaEventRecordWithFlags(e0.cuda_event, stream.cuda_stream, 1)  # cudaEventRecordExternal
                for i in range(count):
                    fn(i)
                rt.cudaEventRecordWithFlags(e1.cuda_event, stream.cuda_stream, 1)
        torch.cuda.current_stream().wait_stream(stream)
        torch.cuda.synchronize()
        # the window holds exactly `count` steps; it is replayed 5 times and the median reported
        # (one short window alone is at the mercy of a single clock / scheduling hiccup)
        samples = []
        for _ in range(5):
            if world > 1:
                torch.distributed.barrier()
            g.replay()
            torch.cuda.synchronize()
            samples.append(e0.elapsed_time(e1))
        return max_over_ranks(float(np.median(samples)), dev)

    def timed(fn, count, chunk_steps=256):
        """Device time of `count` calls of fn (replayed from CUDA graphs), max over ranks."""
        if count < chunk_steps:
            return timed_in_graph(fn, count)
        n_full, rem = divmod(count, chunk_steps)
        gf = graph_of(fn, chunk_steps) if n_full else None
        gr = graph_of(fn, rem) if rem else None
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # a ~100 us device-side spin ahead of the start event: the host submits the
        # graph(s) while the GPU spins, so no host submission gap lands in the window
        torch.cuda._sleep(200_000)
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
        # untimed: bring clocks and the launch path to steady state (~0.2 s of steps) so a short
        # K measures the same per-step time as a long one
        t0 = time.time()
        while time.time() - t0 < 0.2:
            timed(step, 256)
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

    # ---- per-kernel timings, rotated and plain twins, all with the same launch count
    n_k = max(args.steps, 512)
    t_fused = ms_per_step
    t_fr = timed(step, n_k) / n_k
    t_fp = timed(lambda i: fused(sets[i % R], None), n_k) / n_k
    t_k1 = timed(lambda i: k1(sets[i % R]), n_k) / n_k
    t_k2 = timed(lambda i: k2(sets[i % R]), n_k) / n_k
    t_k1p = timed(lambda i: k1(sets[i % R], None), n_k) / n_k
    t_k2p = timed(lambda i: k2(sets[i % R], None), n_k) / n_k
    # row f3 at C2: a learned spec (same signs, an orthogonal R, learned_values) -- the fused learned
    # decode (q T in the kernel's prologue, o T^T before the store: one launch), and the serving
    # step (the new token through the fused learned K1, then that decode).  Same bytes read;
    # the values decoded are not meaningful (the pool was written with the Hadamard spec).
    qm_, rm_ = np.linalg.qr(np.random.default_rng(7).standard_normal((D, D)))
    lspec = RotationSpec(order=ORDER, signs=spec.signs, learned=qm_ * np.sign(np.diag(rm_)), learned_values=True)
    t_k2l = timed(lambda i: k2(sets[i % R], lspec), n_k) / n_k
    t_fl = timed(lambda i: fused(sets[i % R], lspec), n_k) / n_k
    learned_c2 = {"decode_us": round(t_k2l * 1e3, 3), "step_us": round(t_fl * 1e3, 3),
                  "hadamard_decode_us": round(t_k2 * 1e3, 3), "hadamard_step_us": round(t_fused * 1e3, 3),
                  "launches_decode": "one kvr_paged_decode_learned (q T in the prologue, o T^T in the merge)",
                  "launches_step": "the fused learned K1 (store_tc_kernel<LEARNED>, the new token) + the fused learned decode"}
    print(f"[bench] learned R at C2 {learned_c2}", file=sys.stderr, flush=True)
    # restore the rotated token in every set (the plain / learned twins overwrote slot L)
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

    # ---- e2e through the public API with host buffers (rotating over the buffer sets)
    e2e = e2e_api(torch, layout, spec, dev, [st["table"] for st in sets], args, world)

    # ---- verification gather (after timing; NCCL only here)
    if world > 1:  # every rank's sequence (batch shard) gathered on all ranks
        gathered = gather_rows(sets[0]["out"], [1] * world)
        assert gathered.shape[0] == world
    splits = sets[0]["plan"].splits

    # ---- the other BASELINE configs (parity-test cases, reported in `detail`)
    c1 = c1_quantize_store(torch, layout, spec, dev, gen, timed)
    c2v = c2_variants(torch, layout, spec, dev, gen, timed)
    print(f"[bench] C2 variants {c2v}", file=sys.stderr, flush=True)
    print(f"[bench] C1 K1 rot {c1['rot_us']} us plain {c1['plain_us']} (tcgen05 {c1['tcgen05_rot_us']} / "
          f"{c1['tcgen05_plain_us']}); 65536 tok rot {c1['write_65536_tokens']['rot_us']} plain "
          f"{c1['write_65536_tokens']['plain_us']} (mma.sync {c1['write_65536_tokens']['mma_sync_rot_us']}); "
          f"K4 {c1['dequant_us']} us", file=sys.stderr, flush=True)
    print(f"[bench] learned R fused K1 {c1['learned_r_fused']}", file=sys.stderr, flush=True)
    c3 = c4 = c5 = bf = pf = None
    if not args.quick:
        sets.clear()  # free the headline's buffers first
        torch.cuda.empty_cache()
        c3 = c3_sweep(torch, dev, gen, timed)
        print(f"[bench] C3 {[(r['batch'], r['us'], r['frac']) for r in c3]}", file=sys.stderr, flush=True)
        c5 = c5_long(torch, dev, gen, timed, world, rank)
        print(f"[bench] C5 {[(r['ctx'], r['rot_order'], r['us'], r['frac']) for r in c5]}", file=sys.stderr, flush=True)
        c4 = c4_llama70b(torch, dev, gen, timed, world, rank)
        print(f"[bench] C4 step {c4['step_us']} us, {c4['tok_per_s_per_gpu']} tok/s/GPU", file=sys.stderr, flush=True)
        bf = bf16_pool_decode(torch, dev, gen, timed, round(t_k2 * 1e3, 3), c3[1]["us"] if len(c3) > 1 else None)
        print(f"[bench] BF16 pool decode {bf}", file=sys.stderr, flush=True)
        pf = prefill_sweep(torch, dev, gen, timed)
        print(f"[bench] prefill write sweep {[(r['tokens'], r['rotk_us'], r['plain_us'], r['dequant_us']) for r in pf['rows']]}",
              file=sys.stderr, flush=True)

    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu:  # the CPU legs: rank 0 at N = 1 only, after timing
        parity = parity_checks(torch, dev)  # the oracle as the checker (never timed, never shipped)
        print(f"[bench] parity {parity}", file=sys.stderr, flush=True)
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
        "config": headline_config(world),
        "timing": {"decode_splits": splits, "buffer_sets": R, "buffer_set_MB": round(step_bytes(Lstep) / 1e6, 1),
                   "method": "K steps replayed from CUDA graphs, CUDA events on the launching stream after a "
                             "device-side spin that covers the host's graph submission, max over ranks"},
        "roofline": {"bound": "hbm", "kernel": ("decode_tma_kernel (one kvr_decode_step: fused append + split-K "
                                                "decode + inline split merge by the last CTA)") if splits <= 32 else
                     "decode_tma_kernel + decode_merge_kernel (fused append + split-K decode, then the split merge)",
                     "achieved": round(ach, 1), "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": round(ach / peak, 4), "traffic": traffic, "algorithmic_bytes": dbytes,
                     "avg_launch_us": round(t_fused * 1e3, 3)},
        "cpu_baseline": cpu,
        "parity": parity,
        "e2e": e2e,
        # per step: the fused decode kernel (+ the split-merge kernel above 32 splits;
        # 2..8 merge in a cluster, 9..32 inline in the last CTA)
        "gpu_launches": args.steps * (2 if splits > 32 else 1),
        "clocks": clocks,
        "detail": {
            "k1_write_1tok_us": round(t_k1 * 1e3, 3), "k1_plain_1tok_us": round(t_k1p * 1e3, 3),
            "k2_decode_us": round(t_k2 * 1e3, 3), "k2_plain_us": round(t_k2p * 1e3, 3),
            "k2_overhead_vs_plain": round(t_k2 / t_k2p - 1.0, 4),
            "twin_launches": n_k,
            "fused_step_us": round(t_fr * 1e3, 3), "fused_step_plain_us": round(t_fp * 1e3, 3),
            "fused_step_overhead_vs_plain": round(t_fr / t_fp - 1.0, 4),
            "c1_quantize_store": c1,
            "c2_learned_r": learned_c2,
            "c2_input_variants": c2v,
            "c3_concurrency_sweep": c3,
            "c4_llama70b": c4,
            "c5_long_context_1kv_per_gpu": c5,
            "bf16_pool_decode": bf,
            "prefill_write_sweep": pf,
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
        for c0 in range(0, L, chunk):  # (c5_shard_check regenerates 1-head data in this order)
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


def kv_profile(torch, kind, n, Hh, Dd, gen, dev):
    """K/V rows (bf16) of the reference harness's profiles (harness.py:82-176), generated on
    the device: 'outlier' -- Rademacher bulk with one fixed +-27 hot channel per head;
    'correlated' -- Student-t(4)/sqrt(2) rows through a dense rank-4 mixing, two x100 channels."""
    if kind == "outlier":
        x = torch.where(torch.rand((n, Hh, Dd), generator=gen, device=dev) < 0.5, -1.0, 1.0)
        ch = torch.randint(0, Dd, (Hh,), generator=gen, device=dev)
        sgn = torch.where(torch.rand((n, Hh), generator=gen, device=dev) < 0.5, -27.0, 27.0)
        x[:, torch.arange(Hh, device=dev), ch] = sgn
    else:
        z = torch.randn((n, Hh, Dd), generator=gen, device=dev)
        chi = sum(torch.randn((n, Hh, 1), generator=gen, device=dev) ** 2 for _ in range(4)) / 4.0
        x = z / chi.sqrt() / 2.0 ** 0.5
        a = torch.randn((Dd, 4), generator=gen, device=dev)
        b = torch.randn((4, Dd), generator=gen, device=dev)
        mix = torch.eye(Dd, device=dev) + (0.75 / (4 * Dd) ** 0.5) * (a @ b)
        x = x @ mix.T
        ch = torch.randperm(Dd, generator=gen, device=dev)[:2]
        x[:, :, ch] *= 100.0
    return x.to(torch.bfloat16)


def c2_variants(torch, layout, spec, dev, gen, timed):
    """the C2 fused step on the harness's outlier and correlated K/V
    profiles, and on a pool whose pages are randomly permuted (block tables point all over
    the pool instead of in allocation order)."""
    from paper_2604_19157_b200 import PageTable

    P, Hh, Dd, L = layout.page_tokens, layout.num_kv_heads, layout.head_dim, CTX
    res = {}
    for kind in ("outlier", "correlated", "gaussian_shuffled_pages"):
        tables = []
        for _ in range(4):
            t = PageTable(layout, num_pages=-(-(L + 1) // P) + 1, device=dev)
            t.create_sequence(0)
            slots = torch.from_numpy(t.alloc.reserve(0, L)).to(dev)
            for c0 in range(0, L, 8192):
                n = min(8192, L - c0)
                if kind == "gaussian_shuffled_pages":
                    k = torch.randn((n, Hh, Dd), generator=gen, device=dev).to(torch.bfloat16)
                    v = torch.randn((n, Hh, Dd), generator=gen, device=dev).to(torch.bfloat16)
                else:
                    k, v = kv_profile(torch, kind, n, Hh, Dd, gen, dev), kv_profile(torch, kind, n, Hh, Dd, gen, dev)
                t.store_slots(k, v, slots[c0:c0 + n], spec)
            if kind == "gaussian_shuffled_pages":  # move every page to a random physical place
                pages = t.alloc.seq_pages[0]
                perm = torch.randperm(t.num_pages, generator=gen, device=dev)
                new = t.pool.clone()
                new[perm[torch.tensor(pages, device=dev)]] = t.pool[torch.tensor(pages, device=dev)]
                t.pool.copy_(new)
                t.alloc.seq_pages[0] = [int(x) for x in perm[torch.tensor(pages, device=dev)].cpu()]
                used = set(t.alloc.seq_pages[0])
                t.alloc.free = sorted(p for p in range(t.num_pages) if p not in used)
            tables.append(t)
        r = decode_case(torch, dev, tables, spec, timed, fused=True, n=256, gen=gen)
        res[kind] = {"us": r["us"], "plain_us": r["plain_us"], "frac": r["frac"],
                     "overhead_vs_plain": r["overhead_vs_plain"]}
        del tables
    return res


# PAPER.md Table (prefill kernel profiling, Qwen3-32B on 2x H100, tp = 2, one layer): the
# _quantized_set_kv_int4_kernel (INT4, INT4-Fused-RotateK) and flatten_dequant rows, us
PAPER_PREFILL = {8192: (22.05, 29.44, 7.65, 21.63), 16384: (39.04, 52.13, 15.87, 38.69),
                 32768: (74.11, 98.18, 33.18, 75.39), 65536: (135.87, 212.32, 69.22, 165.47),
                 131072: (253.47, 402.33, 137.34, 313.79)}


def prefill_sweep(torch, dev, gen, timed):
    """Row f2: the prefill-sized write (K1) and flatten-dequant (K4) at 8k-128k tokens on the
    paper's prefill shape (Qwen3-32B at tp = 2: 4 kv heads x 128 per GPU), rotated K only
    ("Fused-RotateK", Targets.KEYS_ONLY) and plain, beside the paper's H100 numbers
    (other hardware: context, not a target).  Each size rotates over independent tables,
    inputs and outputs totalling > 2x L2."""
    import ctypes

    from paper_2604_19157_b200 import HeadLayout, PageTable, RotationSpec, Targets, _kernels, _lib, make_signs
    Hq, Dq = 4, 128
    lay = HeadLayout(num_q_heads=32, num_kv_heads=Hq, head_dim=Dq, rot_order=128, page_tokens=P)
    spk = RotationSpec(order=128, signs=make_signs(0, 0, Dq, 128), targets=Targets.KEYS_ONLY)
    peak, _ = hbm_peak()
    rows = []
    for n_tok in sorted(PAPER_PREFILL):
        # R independent sets (table, inputs, outputs) rotate so that the timed loop touches > 2x L2:
        # no launch reads L2-warm inputs or rewrites L2-resident output lines
        set_bytes = n_tok * (4 * Hq * Dq * 2 + 2 * Hq * (Dq + 10) + 8)
        R = max(2, -(-300_000_000 // set_bytes))
        sets = []
        for _ in range(R):
            t = PageTable(lay, num_pages=n_tok // P, device=dev)
            t.create_sequence(0)
            t.alloc.plan([0] * n_tok)
            slots = torch.arange(n_tok, dtype=torch.int64, device=dev)
            k = torch.randn((n_tok, Hq, Dq), generator=gen, device=dev).to(torch.bfloat16)
            v = torch.randn((n_tok, Hq, Dq), generator=gen, device=dev).to(torch.bfloat16)
            bt, lens, ml = t.block_table([0])
            ko = torch.empty((1, n_tok, Hq, Dq), dtype=torch.bfloat16, device=dev)
            sets.append((t, slots, k, v, bt, lens, ml, ko, torch.empty_like(ko)))
        n = 16

        def wr(i, sp):
            t, slots, k, v = sets[i % R][:4]
            t.store_slots(k, v, slots, sp)
        t_r = timed(lambda i: wr(i, spk), n) / n
        t_p = timed(lambda i: wr(i, None), n) / n

        def deq(i):
            t, _, _, _, bt, lens, ml, ko, vo = sets[i % R]
            _lib.check(_lib.lib().kvr_dequantize_pages(ctypes.byref(t.desc), _kernels.ptr(bt), bt.shape[1],
                                                       _kernels.ptr(lens), 1, ml, _kernels.ptr(ko), _kernels.ptr(vo),
                                                       _lib.KVR_BF16, _kernels.stream_ptr()))
        t_d = timed(deq, n) / n
        wb = n_tok * (2 * Hq * Dq * 2 + Hq * (Dq + 10) + 8)
        db = n_tok * (Hq * (Dq + 10) + 2 * Hq * Dq * 2)
        pp = PAPER_PREFILL[n_tok]
        rows.append({"tokens": n_tok, "rotk_us": round(t_r * 1e3, 2), "plain_us": round(t_p * 1e3, 2),
                     "dequant_us": round(t_d * 1e3, 2),
                     "write_frac": round(wb / (t_r * 1e-3) / 1e9 / peak, 4),
                     "dequant_frac": round(db / (t_d * 1e-3) / 1e9 / peak, 4),
                     "paper_h100_int4_us": pp[0], "paper_h100_fused_rotatek_us": pp[1],
                     "paper_h100_dequant_int4_us": pp[2], "paper_h100_dequant_rotatek_us": pp[3], "sets": R})
        del sets
        torch.cuda.empty_cache()
    return {"shape": "Qwen3-32B tp=2 prefill: 4 kv heads x 128 per GPU, page 16, bf16 in, one layer",
            "rotation": "block Hadamard order 128 on K (Targets.KEYS_ONLY), as the paper's Fused-RotateK",
            "paper_source": "PAPER.md prefill kernel profiling table (2x H100, SGLang)", "rows": rows}


def bf16_pool_decode(torch, dev, gen, timed, int4_c2_us, int4_c3_b16_us):
    """the BF16 baseline pool (raw bf16 rows, cache.py:115-118) decoded by the
    tensor-core BF16 kernel at the C2 shape and at C3 B = 16 x 8k, beside the INT4 decode."""
    from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable
    from paper_2604_19157_b200.cache import BF16

    lay = HeadLayout(num_q_heads=NQ, num_kv_heads=H, head_dim=D, rot_order=ORDER, page_tokens=P)
    res = {}
    peak, _ = hbm_peak()
    for name, B, L, int4_us in (("c2_b1_32k", 1, CTX, int4_c2_us), ("c3_b16_8k", 16, 8192, int4_c3_b16_us)):
        R = max(2, -(-300_000_000 // (B * L * H * D * 4)))  # > 2x L2 of rotating tables
        tables = []
        for _ in range(R):
            t = PageTable(lay, precision=BF16, num_pages=B * (-(-L // P)), device=dev)
            for b in range(B):
                t.create_sequence(b)
                sl = torch.from_numpy(t.alloc.reserve(b, L)).to(dev)
                for c0 in range(0, L, 8192):
                    n = min(8192, L - c0)
                    t.store_slots(torch.randn((n, H, D), generator=gen, device=dev).to(torch.bfloat16),
                                  torch.randn((n, H, D), generator=gen, device=dev).to(torch.bfloat16), sl[c0:c0 + n], None)
            tables.append(t)
        plans = [DecodePlan(t, list(range(B))) for t in tables]
        q = torch.randn((B, NQ, D), generator=gen, device=dev).to(torch.bfloat16)
        outs = [torch.empty((B, NQ, D), dtype=torch.float32, device=dev) for _ in tables]
        us = timed(lambda i: plans[i % R].run(q, None, out=outs[i % R]), 256) / 256 * 1e3
        byts = B * (L * H * D * 4 + -(-L // P) * 4 + NQ * D * (2 + 4))
        res[name] = {"us": round(us, 3), "GBps": round(byts / (us * 1e-6) / 1e9, 1),
                     "frac": round(byts / (us * 1e-6) / 1e9 / peak, 4), "splits": plans[0].splits,
                     "int4_decode_us": int4_us, "int4_speedup": round(us / int4_us, 3) if int4_us else None,
                     "kernel": "decode_bf16_kernel (mma.sync bf16, SW128 TMA cells, split-K)"}
        del tables, plans
    return res


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


def c4_llama70b(torch, dev, gen, timed, world, rank):
    """BASELINE configs[3]: Llama-3-70B KV geometry (8 kv heads, 64 q heads, d 128),
    128 sequences x 16k context sharded by sequence: 128 / N per GPU.  One step = the
    fused append + decode of all 80 layers.  The 80 layer caches are resident when they
    fit a 64 GB budget (N >= 4); otherwise the step cycles its 80 launches over the
    caches that fit (each >= 0.58 GB, far above the 126 MB L2, so no launch reads a
    warm cache) -- stated in the result."""
    from paper_2604_19157_b200 import HeadLayout, RotationSpec, make_signs
    from paper_2604_19157_b200.shard import block_range

    layers, B_total, L = 80, 128, 16384
    mine = block_range(B_total, world, rank)
    B = len(mine)
    layout = HeadLayout(num_q_heads=64, num_kv_heads=8, head_dim=D, rot_order=ORDER, page_tokens=P)
    spec = RotationSpec(order=ORDER, signs=make_signs(0, 0, D, ORDER))
    per_layer = B * L * TOK_BYTES
    resident = max(2, min(layers, int(64e9 // per_layer)))
    base = build_table(torch, layout, spec, dev, gen, B, L)
    tables = [base] + [clone_table(torch, base) for _ in range(resident - 1)]
    r = decode_case(torch, dev, tables, spec, timed, fused=True, n=layers * 4, gen=gen)
    step_us = r["us"] * layers
    res = {"layers": layers, "sequences_total": B_total, "sequences_per_gpu": B, "ctx": L, "q_heads": 64,
           "kv_heads": 8, "layer_step_us": r["us"], "layer_plain_us": r["plain_us"], "step_us": round(step_us, 1),
           "tok_per_s_per_gpu": round(B / (step_us * 1e-6), 1),
           "tok_per_s_all_gpus": round(world * B / (step_us * 1e-6), 1), "GBps": r["GBps"], "frac": r["frac"],
           "overhead_vs_plain": r["overhead_vs_plain"], "splits": r["splits"],
           "bytes_per_step": r["algorithmic_bytes"] * layers, "resident_layer_caches": resident,
           "note": (f"{B} of the 128 sequences on this GPU; each step runs all 80 fused append+decode launches"
                    + ("" if resident == layers else f", cycling over {resident} resident layer caches of "
                       f"{per_layer / 1e9:.2f} GB (80 x {per_layer / 1e9:.2f} GB does not fit one GPU)"))}
    del tables, base
    torch.cuda.empty_cache()
    return res


def c5_long(torch, dev, gen, timed, world=1, rank=0):
    """BASELINE configs[4]: one request at 128k / 1M tokens, KV heads sharded 8 ways:
    each rank holds 1 kv head + its 4 q heads (rank r = head r), split-K decode,
    Hadamard order 64 / 128.  With N > 1 ranks the 128k outputs of all ranks are
    gathered after timing (NCCL) and rank 0 checks them against one decode of an
    N-head table built from the same per-head data."""
    from paper_2604_19157_b200 import HeadLayout, RotationSpec, make_signs

    out = []
    for L in (131072, 1048576):
        for order in (128, 64):
            layout = HeadLayout(num_q_heads=4, num_kv_heads=1, head_dim=D, rot_order=order, page_tokens=P)
            spec = RotationSpec(order=order, signs=make_signs(0, 0, D, order))
            reps = max(2, -(-300_000_000 // (L * (D + 10))))
            hg = torch.Generator(device=dev)
            hg.manual_seed(9000 + 97 * rank + order + L)  # this head's data
            base = build_table(torch, layout, spec, dev, hg, 1, L)
            tables = [base] + [clone_table(torch, base) for _ in range(reps - 1)]
            res = decode_case(torch, dev, tables, spec, timed, gen=hg, n=128)
            if world > 1 and L == 131072 and order == 128:
                res["shard_check_rel_err"] = c5_shard_check(torch, dev, layout, spec, base, world, rank, L, order)
            out.append(res)
            del tables, base
            torch.cuda.empty_cache()
    return out


def c5_shard_check(torch, dev, layout, spec, table, world, rank, L, order):
    """Gather every rank's head output (all_gather over NCCL) and compare on rank 0
    with a single-GPU decode of the N-head table of the same data."""
    from paper_2604_19157_b200 import DecodePlan, HeadLayout
    from paper_2604_19157_b200.shard import gather_rows

    qg = torch.Generator(device=dev)
    qg.manual_seed(77 + rank)
    q = torch.randn((1, 4, D), generator=qg, device=dev).to(torch.bfloat16)
    mine = DecodePlan(table, [0]).run(q, spec)
    allq = gather_rows(q.reshape(4, D), [4] * world).reshape(1, 4 * world, D)
    allo = gather_rows(mine.reshape(4, D), [4] * world).reshape(1, 4 * world, D)
    if rank != 0:
        return None
    full = HeadLayout(num_q_heads=4 * world, num_kv_heads=world, head_dim=D, rot_order=order, page_tokens=P)
    heads = []
    for r in range(world):  # rebuild every head's data from its rank's seed
        hg = torch.Generator(device=dev)
        hg.manual_seed(9000 + 97 * r + order + L)
        heads.append(hg)
    from paper_2604_19157_b200 import PageTable
    t = PageTable(full, num_pages=-(-L // P), device=dev)
    t.create_sequence(0)
    slots = torch.from_numpy(t.alloc.reserve(0, L)).to(dev)
    for c0 in range(0, L, 16384):
        n = min(16384, L - c0)
        ks, vs = [], []
        for hg in heads:
            ks.append(torch.randn((n, 1, D), generator=hg, device=dev).to(torch.bfloat16))
            vs.append(torch.randn((n, 1, D), generator=hg, device=dev).to(torch.bfloat16))
        t.store_slots(torch.cat(ks, 1), torch.cat(vs, 1), slots[c0:c0 + n], spec)
    ref = DecodePlan(t, [0]).run(allq, spec)
    return float((allo - ref).abs().max() / ref.abs().max())


def c1_quantize_store(torch, layout, spec, dev, gen, timed):
    """configs[0] shape on the GPU: 4096 tokens x 8 kv heads, order 128, bf16 in."""
    from paper_2604_19157_b200 import PageTable

    from paper_2604_19157_b200 import _lib as _L

    def make_sets(n_tok, R):
        sets = []
        for r in range(R):
            t = PageTable(layout, num_pages=n_tok // P, device=dev)
            t.create_sequence(0)
            slots = torch.arange(n_tok, dtype=torch.int64, device=dev)
            t.alloc.plan([0] * n_tok)
            k = torch.randn((n_tok, H, D), generator=gen, device=dev).to(torch.bfloat16)
            v = torch.randn((n_tok, H, D), generator=gen, device=dev).to(torch.bfloat16)
            sets.append((t, k, v, slots))
        return sets

    def k1_us(sets, n):
        R = len(sets)
        t_r = timed(lambda i: sets[i % R][0].store_slots(sets[i % R][1], sets[i % R][2], sets[i % R][3], spec), n) / n
        t_p = timed(lambda i: sets[i % R][0].store_slots(sets[i % R][1], sets[i % R][2], sets[i % R][3], None), n) / n
        return t_r, t_p

    n_tok, R = 4096, 8
    sets = make_sets(n_tok, R)
    n = 256
    t_rot, t_pl = k1_us(sets, n)  # the default dispatch (mma.sync kernel at this size)
    _L.lib().kvr_debug_set_k1_impl(2)  # A/B: the tcgen05 kernel forced at this size
    try:
        c_rot, c_pl = k1_us(sets, n)
    finally:
        _L.lib().kvr_debug_set_k1_impl(0)
    byts = n_tok * WRITE_BYTES_PER_TOKEN
    peak, _ = hbm_peak()
    # the 65,536-token bulk (prefill-sized) write, both kernels
    big_n = 65536
    big = make_sets(big_n, 2)
    b_rot, b_pl = k1_us(big, 64)  # default dispatch: the tcgen05 kernel at this size
    _L.lib().kvr_debug_set_k1_impl(1)
    try:
        bm_rot, bm_pl = k1_us(big, 64)
    finally:
        _L.lib().kvr_debug_set_k1_impl(0)
    # row f3: the learned R fused into the tcgen05 K1 (T = diag(s) H_blk R as three bf16 parts, 24 MMAs
    # of M128 N128 K16 per tile) vs the unfused route (f64 FWHT + cuBLAS DGEMM, then the exact store)
    import numpy as _np

    from paper_2604_19157_b200 import RotationSpec as _RS
    from paper_2604_19157_b200.rotation import learned_on, learned_store_operands
    qm, rm = _np.linalg.qr(_np.random.default_rng(7).standard_normal((D, D)))
    lspec = _RS(order=spec.order, signs=spec.signs, learned=qm * _np.sign(_np.diag(rm)), learned_values=True)
    learned_store_operands(lspec, layout, dev)
    learned_on(lspec, dev)

    def kl_us(sets_, n_, exact=False):
        R_ = len(sets_)
        return timed(lambda i: sets_[i % R_][0].store_slots(sets_[i % R_][1], sets_[i % R_][2], sets_[i % R_][3], lspec,
                                                          exact=exact), n_) / n_

    l_small, l_small_unf = kl_us(sets, n), kl_us(sets, 32, exact=True)
    l_big, l_big_unf = kl_us(big, 64), kl_us(big, 8, exact=True)
    os.environ["KVR_K1L_FAST"] = "1"  # opt-in fast mode: flagged words under the kernel's own (s, z)
    try:
        l_small_fast, l_big_fast = kl_us(sets, n), kl_us(big, 64)
    finally:
        del os.environ["KVR_K1L_FAST"]
    learned_line = {"kernel": "store_tc_kernel<LEARNED> (tcgen05.mma M128 N128 K16 x 24 per tile, T in shared memory)",
                    "c1_us": round(l_small * 1e3, 3), "c1_GBps": round(byts / (l_small * 1e-3) / 1e9, 1),
                    "c1_frac": round(byts / (l_small * 1e-3) / 1e9 / peak, 4),
                    "c1_unfused_us": round(l_small_unf * 1e3, 2),
                    "t65536_us": round(l_big * 1e3, 2),
                    "t65536_GBps": round(big_n * WRITE_BYTES_PER_TOKEN / (l_big * 1e-3) / 1e9, 1),
                    "t65536_frac": round(big_n * WRITE_BYTES_PER_TOKEN / (l_big * 1e-3) / 1e9 / peak, 4),
                    "t65536_unfused_us": round(l_big_unf * 1e3, 2),
                    "mode": "exact rows (default): a row with a code near a boundary is redone whole in f64 under "
                            "the reference's (s, z) -- codes identical to the f64 reference",
                    "fast_mode_c1_us": round(l_small_fast * 1e3, 3), "fast_mode_t65536_us": round(l_big_fast * 1e3, 2),
                    "fast_mode": "KVR_K1L_FAST=1: flagged words under the kernel's own (s, z); ~1.5e-6 of codes one "
                                 "step off the reference",
                    "t65536_vs_hadamard_only": round(l_big / b_rot - 1.0, 4)}
    del big
    bb = big_n * WRITE_BYTES_PER_TOKEN
    big_line = {"tokens": big_n, "algorithmic_bytes": bb, "rot_us": round(b_rot * 1e3, 2), "plain_us": round(b_pl * 1e3, 2),
                "rot_GBps": round(bb / (b_rot * 1e-3) / 1e9, 1), "rot_frac": round(bb / (b_rot * 1e-3) / 1e9 / peak, 4),
                "overhead_vs_plain": round(b_rot / b_pl - 1.0, 4),
                "kernel": "store_tc_kernel (tcgen05.mma M128 N16 K16, TMEM accumulators, TMA ring; the default here)",
                "mma_sync_rot_us": round(bm_rot * 1e3, 2), "mma_sync_plain_us": round(bm_pl * 1e3, 2)}
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
            "overhead_vs_plain": round(t_rot / t_pl - 1.0, 4),
            "kernel": "store_mma_kernel (mma.sync; the default below ~4 tiles of 128 rows per SM)",
            "tcgen05_rot_us": round(c_rot * 1e3, 3), "tcgen05_plain_us": round(c_pl * 1e3, 3),
            "write_65536_tokens": big_line, "learned_r_fused": learned_line}


def e2e_api(torch, layout, spec, dev, tables, args, world):
    """Public-API step with host buffers: every step allocates the new token's slot
    (host bookkeeping), copies q and the new K/V from pinned host memory with the
    slot / length metadata, runs the fused append + decode (DecodePlan.step), and the
    kernel writes the output into a pinned host tensor.  The steps rotate over the
    buffer sets' tables (> 2x L2), so no step reads L2-warm KV."""
    from paper_2604_19157_b200 import DecodePlan

    steps = min(max(args.steps, 256), 1000)  # a separate, bounded measurement (not the K of the headline)
    R = len(tables)
    warm = 2 * R * DecodePlan._RING  # every (plan, staging slot) graph is captured before the timed steps
    kh = torch.randn((1, H, D)).to(torch.bfloat16).pin_memory()
    vh = torch.randn((1, H, D)).to(torch.bfloat16).pin_memory()
    qh = torch.randn((1, NQ, D)).to(torch.bfloat16).pin_memory()
    oh = torch.empty((1, NQ, D), dtype=torch.float32).pin_memory()
    saved = [(list(t.alloc.free), t.alloc.seq_len[0], list(t.alloc.seq_pages[0])) for t in tables]
    per_plan = -(-(steps + warm) // R) + 8
    plans = [DecodePlan(t, [0], extra_tokens=per_plan) for t in tables]
    i = [0]

    def one():
        plans[i[0] % R].step(qh, kh, vh, spec, out=oh, graph=True)
        i[0] += 1

    for _ in range(warm):
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
    L = max(t.alloc.seq_len[0] for t in tables)
    for t, (free, ln, pages) in zip(tables, saved):  # roll the tables back
        t.alloc.free = free
        t.alloc.seq_len[0] = ln
        t.alloc.seq_pages[0] = pages
    byts = step_bytes(L)
    return {"value": round(world * byts / (ms * 1e-3) / 1e9, 2), "unit": "GB/s", "ms_per_step": round(ms, 4),
            "h2d_bytes_per_step": kh.numel() * 2 + vh.numel() * 2 + qh.numel() * 2 + 12,  # + slot id, length
            "d2h_bytes_per_step": oh.numel() * 4,
            "api": "DecodePlan.step(graph=True) (fused append + decode) with pinned host buffers",
            "steps": steps, "tables": R, "timing": "max(CUDA events, host wall clock) over the steps"}


def parity_checks(torch, dev):
    """Parity of the timed kernels on this box, with the oracle as the checker (after
    timing): K1 on the C1 shape (4,096 tokens x 8 heads, K & V rotated, Gaussian bf16)
    -- nibble, zero-point and scale mismatch counts vs the reference arithmetic -- and
    the C2 fused step's max relative error vs an oracle-quantised decode."""
    from oracle import kvrot_oracle as O
    from paper_2604_19157_b200 import DecodePlan, HeadLayout, PageTable, RotationSpec, make_signs

    layout = HeadLayout(num_q_heads=NQ, num_kv_heads=H, head_dim=D, rot_order=ORDER, page_tokens=P)
    spec = RotationSpec(order=ORDER, signs=make_signs(0, 0, D, ORDER))
    g = torch.Generator(device=dev)
    g.manual_seed(4242)
    res = {"checker": "oracle/kvrot_oracle.py (numpy restatement of the reference, pinned to its goldens)"}
    # -- K1 at C1
    n_tok = 4096
    t = PageTable(layout, num_pages=n_tok // P, device=dev)
    t.create_sequence(0)
    k = torch.randn((n_tok, H, D), generator=g, device=dev).to(torch.bfloat16)
    v = torch.randn((n_tok, H, D), generator=g, device=dev).to(torch.bfloat16)
    t.append_batch([0] * n_tok, k, v, spec=spec)
    rec = t.page_records(t.sequence_pages(0))
    cells = P * H
    f = {}
    off = 0
    for name, nb, dt in (("k_payload", cells * D // 2, np.uint8), ("v_payload", cells * D // 2, np.uint8),
                         ("k_scale", cells * 4, np.float32), ("k_zp", cells, np.uint8),
                         ("v_scale", cells * 4, np.float32), ("v_zp", cells, np.uint8)):
        f[name] = rec[:, off:off + nb].copy().view(dt).reshape(-1, nb // cells // np.dtype(dt).itemsize)
        off += nb
    k1 = {}
    for side, x in (("k", k), ("v", v)):
        rows = x.double().cpu().numpy().reshape(-1, D)
        p_, s_, z_ = O.quantize_rows(O.rotate_rows(rows, ORDER, spec.signs))
        ours_p = f[f"{side}_payload"].reshape(-1, D // 2)
        x_ = ours_p ^ p_
        k1[side] = {"rows": int(rows.shape[0]),
                    "nibble_mismatches": int(np.count_nonzero(x_ & 0x0F) + np.count_nonzero(x_ & 0xF0)),
                    "zp_mismatches": int(np.count_nonzero(f[f"{side}_zp"].reshape(-1) != z_)),
                    "scale_mismatches": int(np.count_nonzero(f[f"{side}_scale"].reshape(-1).view(np.uint32)
                                                             != s_.view(np.uint32)))}
    res["c1_k1_fast_rotated"] = k1
    # -- C2 fused step
    t2 = PageTable(layout, num_pages=CTX // P + 2, device=dev)
    t2.create_sequence(0)
    slots = torch.from_numpy(t2.alloc.reserve(0, CTX)).to(dev)
    ks, vs = [], []
    for c0 in range(0, CTX, 8192):
        kc = torch.randn((8192, H, D), generator=g, device=dev).to(torch.bfloat16)
        vc = torch.randn((8192, H, D), generator=g, device=dev).to(torch.bfloat16)
        t2.store_slots(kc, vc, slots[c0:c0 + 8192], spec)
        ks.append(kc.double().cpu().numpy())
        vs.append(vc.double().cpu().numpy())
    kn = torch.randn((1, H, D), generator=g, device=dev).to(torch.bfloat16)
    vn = torch.randn((1, H, D), generator=g, device=dev).to(torch.bfloat16)
    q = torch.randn((1, NQ, D), generator=g, device=dev).to(torch.bfloat16)
    out = DecodePlan(t2, [0], extra_tokens=1).step(q, kn, vn, spec)
    kk = np.concatenate(ks + [kn.double().cpu().numpy()]).reshape(-1, D)
    vv = np.concatenate(vs + [vn.double().cpu().numpy()]).reshape(-1, D)
    kh = O.dequantize_rows(*O.quantize_rows(O.rotate_rows(kk, ORDER, spec.signs)), D).reshape(-1, H, D)
    vh = O.dequantize_rows(*O.quantize_rows(O.rotate_rows(vv, ORDER, spec.signs)), D).reshape(-1, H, D)
    ref = O.decode_flat(O.rotate_rows(q[0].double().cpu().numpy(), ORDER, spec.signs), kh, vh, G)
    ref = O.unrotate_rows(ref, ORDER, spec.signs)
    got = out[0].double().cpu().numpy()
    res["c2_fused_step_max_rel_err"] = float(np.abs(got - ref).max() / np.abs(ref).max())
    res["c2_tolerance"] = "1e-3 x max|ref| (north star)"
    return res


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


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform

    return platform.processor() or "unknown"


def _c1_kernel_rows(n_tok=1024, seed=0):
    rng = np.random.default_rng(seed)
    from oracle import kvrot_oracle as O

    k = rng.standard_normal((n_tok * H, D))
    v = rng.standard_normal((n_tok * H, D))
    return O, k, v


def _c1_kernels_once(args):
    """One worker's share of the C1 kernel leg: fwht_rows + quantize_rows on K and V
    rows (the reference's compiled kernels when oracle/_ref is built)."""
    n_tok, seed = args
    O, k, v = _c1_kernel_rows(n_tok, seed)
    _cpu_kernels()
    signs = O.make_signs(0, 0, D, ORDER)
    t0 = time.perf_counter()
    for x in (k, v):
        y = x * signs
        O.fwht_rows(y, ORDER)
        O.quantize_rows(y)
    return time.perf_counter() - t0


def cpu_c1_kernel_legs(seconds: float):
    """(i) kernel-level C1 (fwht_rows + quantize_rows, the reference's
    L0 kernels, bench-attn pattern cli.py:388-431) on one core, and (iii) the same work
    sharded over all host cores with a multiprocessing pool; GB/s with K1's algorithmic
    bytes per token."""
    import multiprocessing as mp

    n_tok = 1024
    one = _c1_kernels_once((n_tok, 0))  # warm
    reps = max(1, int(seconds / 2 / max(one, 1e-3)))
    t1 = min(_c1_kernels_once((n_tok, 0)) for _ in range(min(reps, 5)))
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(_c1_kernels_once, [(n_tok, i) for i in range(cores)])  # warm the workers
        t0 = time.perf_counter()
        pool.map(_c1_kernels_once, [(n_tok, i) for i in range(cores * 4)])
        tn = time.perf_counter() - t0
    b = n_tok * WRITE_BYTES_PER_TOKEN
    return {"c1_kernels_1core_GBps": round(b / t1 / 1e9, 5), "c1_kernels_ncore_GBps": round(4 * cores * b / tn / 1e9, 5),
            "ncore_workers": cores,
            "sample": f"{n_tok} tokens x 8 heads (K and V rows) per task: sign flip + fwht_rows + quantize_rows, "
                      f"f64; 1 core best of {min(reps, 5)}, then {4 * cores} tasks over a {cores}-process pool"}


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
    legs = cpu_c1_kernel_legs(min(seconds, 10.0))
    return {"value": round(step_bytes(L + 1) / t / 1e9, 4), "unit": "GB/s", "cores": _cpu_threads(),
            "kind": kind, "cpu_model": cpu_model(),
            "sample": f"{len(times)} full C2 steps (1-token write + decode over {L + 1} tokens) with "
                      f"{_KIND_NOTE[kind]} (numpy/OpenBLAS threads), median {t * 1e3:.1f} ms/step",
            "legs": legs}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm on the host cores (the compiled
    reference kernels in oracle/_ref when built, else the numpy port), same metric and
    config as the GPU arm; rank 0 only.  Each step is a full C2 step (1-token write +
    decode over 32,769 tokens); if K steps would not fit the time budget, the first
    steps that fit are timed and the count is stated."""
    if rank != 0:
        return
    from oracle import kvrot_oracle as O

    kind = _cpu_kernels()
    rng = np.random.default_rng(0)
    signs = O.make_signs(0, 0, D, ORDER)
    budget = 150.0
    seq = CpuOracleSequence(CTX, rng, signs, extra_tokens=args.steps + args.warmup + 16)
    for _ in range(args.warmup):
        seq.step()
    ts = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ts.append(seq.step())
        if time.perf_counter() - t0 > budget:
            break
    ms = float(np.mean(ts)) * 1e3
    val = step_bytes(CTX + 1) / (ms * 1e-3) / 1e9
    line = {
        "impl": "reference", "metric": "quantize-store + INT4 paged-decode HBM GB/s (one serving decode step, "
                                       "% of HBM roofline)",
        "value": round(val, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 (reference numpy arithmetic)", "data": "synthetic (numpy standard normal)",
        "config": headline_config(world),
        "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": _cpu_threads(), "kind": kind,
                         "cpu_model": cpu_model(),
                         "sample": f"{len(ts)} of {args.steps} steps timed, each a 1-token write + decode over "
                                   f"{CTX + 1} tokens, {_KIND_NOTE[kind]}"},
        "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sets", type=int, default=8)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--quick", action="store_true", help="headline + C1 only (skip the C3/C4/C5 detail configs)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch this command under torch.distributed.run
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
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
