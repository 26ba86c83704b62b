"""N > 1 host path on CPU: world_size 2, gloo (no GPU).  Each rank serves its
shard with the numpy oracle (the kernels' stand-in here), the shards are
gathered with the same helpers bench.py uses, and rank 0 checks the result
equals the unsharded computation -- for batch sharding (C3/C4) and kv-head
sharding of one long request (C5)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import kvrot_oracle as O
from paper_2604_19157_b200 import HeadLayout
from paper_2604_19157_b200.shard import block_range, gather_rows, max_over_ranks, shard_heads, shard_sequences

H, G, D, ORDER, P = 4, 2, 32, 32, 8


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    rng = np.random.default_rng(9)
    lens = [5, 17, 9, 12, 1]
    kv = [(rng.standard_normal((L, H, D)), rng.standard_normal((L, H, D))) for L in lens]
    q = rng.standard_normal((len(lens), H * G, D))
    return lens, kv, q, O.make_signs(0, 0, D, ORDER)


def _decode(seq_ids, heads, kv, q, signs):
    """Oracle decode of sequences `seq_ids` restricted to kv heads `heads`."""
    h = list(heads)
    pages = O.OraclePages(len(h) * G, len(h), D, ORDER, P, 64)
    outs = []
    for n, s in enumerate(seq_ids):
        pages.create_sequence(n)
        k, v = kv[s]
        for t in range(k.shape[0]):
            pages.append_token(n, k[t][h], v[t][h], signs=signs)
        qs = q[s][h[0] * G:(h[-1] + 1) * G]
        outs.append(O.decode_step(pages, n, qs, signs=signs))
    return np.stack(outs)


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lens, kv, q, signs = _problem()
        # batch sharding
        mine = shard_sequences(range(len(lens)), world, rank)
        out = torch.from_numpy(_decode(mine, range(H), kv, q, signs))
        counts = [len(block_range(len(lens), world, r)) for r in range(world)]
        full = gather_rows(out, counts)
        # kv-head sharding of request 1 (all of its q heads, split by kv head)
        layout = HeadLayout(num_q_heads=H * G, num_kv_heads=H, head_dim=D, rot_order=ORDER, page_tokens=P)
        local, kvh, qh = shard_heads(layout, world, rank)
        assert local.num_kv_heads == len(kvh) and local.num_q_heads == len(qh)
        part = torch.from_numpy(_decode([1], kvh, kv, q, signs)[0])
        heads_full = gather_rows(part, [len(shard_heads(layout, world, r)[2]) for r in range(world)])
        t = max_over_ranks(float(rank + 1))
        if rank == 0:
            results["batch"] = full.numpy()
            results["heads"] = heads_full.numpy()
            results["tmax"] = t
    finally:
        dist.destroy_process_group()


def test_block_range_partitions():
    for n in (0, 1, 5, 8, 13):
        for world in (1, 2, 3, 8):
            parts = [block_range(n, world, r) for r in range(world)]
            assert [i for p in parts for i in p] == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_world2_gloo_matches_unsharded():
    world = 2
    with mp.Manager() as m:
        results = m.dict()
        mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
        res = dict(results)
    lens, kv, q, signs = _problem()
    want = _decode(range(len(lens)), range(H), kv, q, signs)
    np.testing.assert_array_equal(res["batch"], want)
    np.testing.assert_allclose(res["heads"], want[1], rtol=0, atol=1e-12)
    assert res["tmax"] == 2.0
