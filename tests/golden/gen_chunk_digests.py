"""Writes tests/golden/c4_chunks.csv and c5_chunks.csv: for every 2^28-index
chunk of the BASELINE.json full-size spaces C4 (configs[3]) and C5
(configs[4]), the oracle's survivor count, per-capacity counts and the two
order-dependent digests of the chunk's feasible set (definition: oracle/
me_oracle.h, or_digest).  Calls only oracle/ (test infrastructure); nothing
here comes from the CUDA path.

Chunk c covers flat indices [c * 2^28, min((c + 1) * 2^28, size)) -- the
sweep calls bench.py makes (bench.CHUNK).  Order of work: the C5 sample the
parity test needs (first chunk, the dense chunk 40, every 16th, the last), all
of C4, then the remaining C5 chunks.  Rows are appended as chunks finish, so
the script resumes where a previous run stopped.

  python tests/golden/gen_chunk_digests.py [--threads T] [--only c4|c5-sample|all]
"""
from __future__ import annotations

import argparse
import csv
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

import me_inputs as mi  # noqa: E402
import oracle  # noqa: E402

CHUNK = 1 << 28
FIELDS = ["chunk", "begin", "end", "count", "cap0", "cap1", "cap2", "cap3", "digest_index", "digest_record"]


def c5_sample(n_chunks: int):
    return sorted({0, 40, n_chunks - 1} | set(range(0, n_chunks, 16)))


def done_chunks(path: Path):
    if not path.exists():
        return set()
    with path.open() as fh:
        return {int(r["chunk"]) for r in csv.DictReader(fh)}


def run(name: str, chunks, threads: int, path: Path = None):
    sp = mi.config(name)
    size = oracle.space_size(sp)
    path = path or HERE / f"{name.lower()}_chunks.csv"
    have = done_chunks(path)
    new = not path.exists()
    with path.open("a", newline="") as fh:
        w = csv.writer(fh)
        if new:
            w.writerow(FIELDS)
        for c in chunks:
            if c in have:
                continue
            b, e = c * CHUNK, min(size, (c + 1) * CHUNK)
            t = time.time()
            d = oracle.digest(sp, b, e, CHUNK, threads)[0]
            w.writerow([c, b, e, int(d[0])] + [int(x) for x in d[1:5]] + [f"{int(d[9]):016x}", f"{int(d[10]):016x}"])
            fh.flush()
            print(f"{name} chunk {c}: {int(d[0])} survivors, {time.time() - t:.0f} s", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=oracle.default_threads())
    ap.add_argument("--only", default="all", choices=["c4", "c5-sample", "all", "c5-range"])
    ap.add_argument("--range", default="", help="c5-range: first:last chunks (inclusive)")
    ap.add_argument("--out", default="", help="c5-range: output CSV (default: tests/golden/c5_chunks.csv)")
    a = ap.parse_args()
    if a.only == "c5-range":
        lo, hi = (int(x) for x in a.range.split(":"))
        run("C5", range(lo, hi + 1), a.threads, Path(a.out) if a.out else None)
        return
    n5 = -(-oracle.space_size(mi.config("C5")) // CHUNK)
    n4 = -(-oracle.space_size(mi.config("C4")) // CHUNK)
    if a.only in ("c5-sample", "all"):
        run("C5", c5_sample(n5), a.threads)
    if a.only in ("c4", "all"):
        run("C4", range(n4), a.threads)
    if a.only == "all":
        run("C5", range(n5), a.threads)


if __name__ == "__main__":
    main()
