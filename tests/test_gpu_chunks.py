"""Whole-chunk parity at full size: BASELINE.json configs[3] (C4) and
configs[4] (C5), north star "bit-exact feasible sets vs the oracle on all 5
configs".

Every 2^28-index chunk the golden file holds (tests/golden/c4_chunks.csv: all
of C4; c5_chunks.csv: at least the first chunk, the dense chunk 40, every 16th
and the last -- written by tests/golden/gen_chunk_digests.py, which calls only
oracle/) is swept on the GPU exactly as bench.py sweeps it (one me_plan_sweep
call per chunk, caller columns) and compared by survivor count, per-capacity
counts and the two order-dependent digests of the feasible set (me.h
me_result_digest; the oracle's or_digest computes the same definition
independently).  A dropped, duplicated, reordered or altered survivor
anywhere in a chunk changes a digest."""
import csv
from pathlib import Path

import numpy as np
import pytest

import me_inputs as mi

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"
CHUNK = 1 << 28


def golden(name):
    p = GOLDEN / f"{name.lower()}_chunks.csv"
    if not p.exists():
        return []
    with p.open() as fh:
        rows = list(csv.DictReader(fh))
    out = []
    for r in rows:
        out.append(dict(chunk=int(r["chunk"]), begin=int(r["begin"]), end=int(r["end"]), count=int(r["count"]),
                        caps=[int(r[f"cap{q}"]) for q in range(4)], di=int(r["digest_index"], 16),
                        dr=int(r["digest_record"], 16)))
    return sorted(out, key=lambda r: r["chunk"])


@pytest.fixture(scope="module")
def me():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2411_06465_b200 as me
    torch.cuda.set_device(0)
    return me


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_whole_chunks_match_oracle(me, name):
    import torch
    rows = golden(name)
    if not rows:
        pytest.skip(f"no golden chunks for {name}")
    sp = mi.config(name)
    plan = me.Plan(sp)
    rec = torch.empty(CHUNK * 8, dtype=torch.int64, device="cuda")
    idx = torch.empty(CHUNK, dtype=torch.int64, device="cuda")
    for r in rows:
        b, e = r["begin"], r["end"]
        assert e == min(plan.size, b + CHUNK)
        res = plan.sweep(b, e, mode=me.ME_OUT_RECORDS, out_cols=[rec])
        assert res.status() == 0
        assert res.counts()[0] == r["count"], r["chunk"]
        assert res.cap_counts() == r["caps"], r["chunk"]
        assert res.digest() == (r["di"], r["dr"]), r["chunk"]
        res.free()
        res = plan.sweep(b, e, mode=me.ME_OUT_INDEX, out_cols=[idx])
        assert res.counts()[0] == r["count"] and res.cap_counts() == r["caps"]
        assert res.digest()[0] == r["di"], r["chunk"]
        res.free()
        res = plan.sweep(b, e, mode=me.ME_OUT_COUNT)
        assert res.counts()[0] == r["count"] and res.cap_counts() == r["caps"], r["chunk"]
        res.free()
    if len(rows) == -(-plan.size // CHUNK):
        # all chunks present: the whole feasible set (C4; C5 once the generator
        # has filled every chunk) -- the survivors of a bench step
        res = plan.sweep(0, 0, mode=me.ME_OUT_COUNT)
        assert res.counts()[0] == sum(r["count"] for r in rows)
        assert res.cap_counts() == [sum(r["caps"][q] for r in rows) for q in range(4)]


def test_full_columns_match_oracle_chunks(me):
    """FULL (eight columns) on the first and the dense chunk of C5"""
    import torch
    rows = [r for r in golden("C5") if r["chunk"] in (0, 40)]
    if not rows:
        pytest.skip("no golden chunks")
    plan = me.Plan(mi.config("C5"))
    cols = [torch.empty(CHUNK, dtype=torch.int64, device="cuda") for _ in range(8)]
    for r in rows:
        res = plan.sweep(r["begin"], r["end"], mode=me.ME_OUT_FULL, out_cols=cols)
        assert res.counts()[0] == r["count"]
        assert res.digest() == (r["di"], r["dr"])


def test_whole_space_in_one_call_matches_chunks(me):
    """C4 in one me_plan_sweep call (sub-ranges cut inside the library) gives
    the same feasible set as the chunked calls: the digest of the whole
    result equals the chunk digests merged in order."""
    import torch
    rows = golden("C4")
    plan = me.Plan(mi.config("C4"))
    if len(rows) != -(-plan.size // CHUNK):
        pytest.skip("C4 golden incomplete")
    total = sum(r["count"] for r in rows)
    idx = torch.empty(total, dtype=torch.int64, device="cuda")
    res = plan.sweep(0, 0, mode=me.ME_OUT_INDEX, out_cols=[idx])
    assert res.status() == 0 and res.counts()[0] == total
    M, W = 0xD1B54A32D192ED03, (1 << 64) - 1
    d, n = 0, 0
    for r in rows:
        d = (d + pow(M, n, 1 << 64) * r["di"]) & W
        n += r["count"]
    assert res.digest()[0] == d


def test_digest_matches_oracle_rows_small(me, oracle_mod):
    """the device digest of a small result equals the definition evaluated on
    the oracle's rows"""
    for sp in (mi.config("C3", uneven=1), mi.config("C1")):
        plan = me.Plan(sp)
        idx, rows, n, caps = oracle_mod.sweep(sp, threads=8)
        ref = oracle_mod.digest_of_rows(idx, rows)
        for mode in (me.ME_OUT_RECORDS, me.ME_OUT_FULL):
            assert plan.sweep(mode=mode).digest() == ref
        assert plan.sweep(mode=me.ME_OUT_INDEX).digest() == (ref[0], 0)
        d = oracle_mod.digest(sp, chunk=1 << 40, threads=4)[0]
        assert (int(d[9]), int(d[10])) == ref
        with pytest.raises(me.MEError):
            plan.sweep(mode=me.ME_OUT_COUNT).digest()
