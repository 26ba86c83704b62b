"""Host-side page allocation mirrors the reference PageTable exactly (CPU only)."""

import numpy as np
import pytest

from oracle import kvrot_oracle as O
from paper_2604_19157_b200.cache import PageAllocator, capacity_tokens, page_bytes, token_bytes
from paper_2604_19157_b200.errors import CapacityExceededError, ConfigError, SequenceNotFoundError
from paper_2604_19157_b200.layout import HeadLayout

BIG = HeadLayout(num_q_heads=8, num_kv_heads=8, head_dim=128, rot_order=128)


def test_plan_matches_oracle_page_ids():
    rng = np.random.default_rng(0)
    a = PageAllocator(40, 4)
    ref = O.OraclePages(4, 1, 2, 1, 4, 40)
    for s in range(6):
        a.create(s)
        ref.create_sequence(s)
    seqs = [int(x) for x in rng.integers(0, 6, size=120)]
    slots, fresh = a.plan(seqs)
    for i, s in enumerate(seqs):
        t = ref.seq_len[s]
        ref.append_token(s, np.zeros((1, 2)), np.zeros((1, 2)))
        assert slots[i] == ref.seq_pages[s][t // 4] * 4 + t % 4
    assert a.seq_pages == ref.seq_pages and a.seq_len == ref.seq_len
    assert sorted(fresh) == sorted(p for ps in a.seq_pages.values() for p in ps)


def test_lowest_id_reuse_and_release():
    a = PageAllocator(6, 4)
    a.create(0)
    a.create(1)
    a.plan([0] * 9)
    a.plan([1])
    assert a.release(0) == [0, 1, 2]
    a.create(2)
    a.plan([2])
    assert a.seq_pages[2] == [0]


def test_unplan_restores_state():
    """A step that fails after planning its slots is undone completely: lengths,
    page lists and the free heap are as before (the reference never mutates on a
    rejected append, cache.py:225-233)."""
    a = PageAllocator(8, 4)
    for s in (0, 1, 2):
        a.create(s)
    a.plan([0] * 4 + [1] * 3)
    before = (sorted(a.free), {k: list(v) for k, v in a.seq_pages.items()}, dict(a.seq_len))
    slots, fresh = a.plan([0, 1, 2])  # seq 0 and 2 take fresh pages, seq 1 fills its page
    assert len(fresh) == 2
    a.unplan([0, 1, 2], fresh)
    assert (sorted(a.free), {k: list(v) for k, v in a.seq_pages.items()}, dict(a.seq_len)) == before
    assert a.plan([0, 1, 2])[0].tolist() == slots.tolist()  # same slots again
    fr = a.reserve(2, 9)
    assert a.seq_len[2] == 10


def test_all_or_nothing_on_exhaustion():
    a = PageAllocator(2, 4)
    a.create(0)
    a.plan([0] * 8)
    before = (list(a.free), dict(a.seq_len))
    with pytest.raises(CapacityExceededError):
        a.plan([0, 0])
    assert (list(a.free), dict(a.seq_len)) == before
    with pytest.raises(SequenceNotFoundError):
        a.plan([5])
    with pytest.raises(ConfigError):
        a.create(0)


def test_byte_accounting_frozen():
    # test_cache.py:37-52
    assert token_bytes(BIG, "bf16") == 4096
    assert token_bytes(BIG, "int4") == 1024
    assert token_bytes(BIG, "int4", include_sidecar=True) == 1104
    assert capacity_tokens(1 << 20, BIG, "bf16") == 256
    assert capacity_tokens(1 << 20, BIG, "int4") == 1024
    assert page_bytes(BIG) == 16 * 1104


@pytest.mark.parametrize("lay", [(32, 8, 128, 128, 16), (4, 2, 32, 16, 4), (4, 1, 128, 64, 32), (4, 2, 32, 16, 3)])
def test_cell_layout_round_trip(lay):
    """Device cell layout <-> reference .kvpg page records (cache.py:387-397) is a bijection."""
    from paper_2604_19157_b200.cache import cells_to_records, records_to_cells, page_bytes, record_bytes

    layout = HeadLayout(*lay)
    rec = np.random.default_rng(0).integers(0, 256, size=(5, record_bytes(layout)), dtype=np.uint8)
    cells = records_to_cells(rec, layout)
    assert cells.shape == (5, page_bytes(layout))
    np.testing.assert_array_equal(cells_to_records(cells, layout), rec)
