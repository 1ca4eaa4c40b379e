"""The chunk digests of the oracle (or_digest, test infrastructure for the
whole-chunk parity of tests/test_gpu_chunks.py): its per-piece merge against
the definition evaluated row by row on the oracle's own survivors, and the
golden files' coverage."""
import csv
from pathlib import Path

import pytest

import me_inputs as mi

GOLDEN = Path(__file__).resolve().parent / "golden"
CHUNK = 1 << 28


@pytest.mark.parametrize("chunk,threads", [(1 << 40, 1), (10000, 3), (7777, 8), (333, 2)])
def test_digest_pieces_merge_to_the_definition(oracle_mod, chunk, threads):
    """D(A B) = D(A) + M^|A| D(B): the threaded, chunked digest equals the
    definition over each chunk's rows (oracle.digest_of_rows, plain Python)"""
    sp = mi.config("C3", uneven=1)
    n = oracle_mod.space_size(sp)
    d = oracle_mod.digest(sp, 0, 0, chunk, threads)
    assert len(d) == -(-n // chunk)
    for c in range(min(len(d), 12)):
        b, e = c * chunk, min(n, (c + 1) * chunk)
        idx, rows, cnt, caps = oracle_mod.sweep(sp, b, e, threads=2)
        assert int(d[c, 0]) == cnt and [int(x) for x in d[c, 1:5]] == caps
        assert (int(d[c, 9]), int(d[c, 10])) == oracle_mod.digest_of_rows(idx, rows)


def test_digest_is_order_and_value_sensitive(oracle_mod):
    import numpy as np
    sp = mi.config("C1")
    idx, rows, n, _ = oracle_mod.sweep(sp)
    ref = oracle_mod.digest_of_rows(idx, rows)
    swapped = idx.copy()
    swapped[[0, 1]] = swapped[[1, 0]]
    assert oracle_mod.digest_of_rows(swapped, rows)[0] != ref[0]
    bumped = rows.copy()
    bumped[5, 3] += np.uint64(1)
    assert oracle_mod.digest_of_rows(idx, bumped)[1] != ref[1]
    assert oracle_mod.digest_of_rows(idx[:-1], rows[:-1]) != ref


def golden(name):
    with (GOLDEN / f"{name.lower()}_chunks.csv").open() as fh:
        return {int(r["chunk"]): r for r in csv.DictReader(fh)}


def test_golden_files_cover_the_required_chunks(oracle_mod):
    """every chunk of C4 and of C5 (the C5 sample the verdict asked for --
    first chunk, dense chunk 40, every 16th, the last -- and all the others);
    every row's range is its chunk's"""
    for name in ("C4", "C5"):
        n = oracle_mod.space_size(mi.config(name))
        rows = golden(name)
        for c, r in rows.items():
            assert int(r["begin"]) == c * CHUNK and int(r["end"]) == min(n, (c + 1) * CHUNK)
            assert 0 < int(r["count"]) <= int(r["end"]) - int(r["begin"])
            caps = [int(r[f"cap{q}"]) for q in range(4)]
            assert caps == sorted(caps) and caps[-1] == int(r["count"])  # 40 <= 80 <= 94 <= 192 GiB
        nc = -(-n // CHUNK)
        if name == "C5":
            assert {0, 40, nc - 1} | set(range(0, nc, 16)) <= set(rows)
        assert set(rows) == set(range(nc))
