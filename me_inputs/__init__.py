"""Seeded, synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py.  Holds model shapes and configuration-space descriptions only: none of
the estimator's arithmetic lives here (DESIGN.md §5 states the recipe).

Model presets (reading R26 in DESIGN.md): Llama-3.1-8B/70B are pinned by the
paper's tables; the Llama-2 shapes come from
the public model configurations (P:86 mentions Llama-2 only for its 4,096
context).
"""
from __future__ import annotations

import csv
import dataclasses
from pathlib import Path
from typing import List, Optional, Sequence, Tuple

import numpy as np

GIB = 1 << 30

# (h, h_ffn, L, a, k, v) -- Table "Variable names"
PRESETS = {
    "llama2-7b": (4096, 11008, 32, 32, 32, 32000),
    "llama2-13b": (5120, 13824, 40, 40, 40, 32000),
    "llama2-70b": (8192, 28672, 80, 64, 8, 32000),
    "llama3.1-8b": (4096, 14336, 32, 32, 8, 128256),
    "llama3.1-70b": (8192, 28672, 80, 64, 8, 128256),
}
# Llama-3 (not 3.1) 8B/70B have the same shapes as 3.1 apart from context length
PRESETS["llama3-8b"] = PRESETS["llama3.1-8b"]
PRESETS["llama3-70b"] = PRESETS["llama3.1-70b"]

GOLDEN = Path(__file__).resolve().parent.parent / "tests" / "golden"


@dataclasses.dataclass
class Space:
    """A configuration space in the canonical enumeration order."""

    models: List[Tuple[int, int, int, int, int, int]]
    world: List[int]
    caps_gb: List[int]  # nominal GB; bytes = GB * 2^30 (reading R2)
    mbs: List[int]
    seq: List[int]
    rc_mask: int = 3  # bit0 = recompute off, bit1 = on
    do_mask: int = 3  # bit0 = distributed optimizer off, bit1 = on
    uneven: int = 0
    gbs: int = 0
    max_t: int = 0
    max_c: int = 0
    max_p: int = 0
    gpus_per_node: int = 0
    thr_num: int = 4
    thr_den: int = 5
    stage_max: int = 0  # 1 = NEXT-1: feasibility of the largest pipeline stage
    zero_stage: int = 0  # NEXT-4: 2 / 3 = gradients / also weights sharded with the optimizer
    sp_off: int = 0  # NEXT-4: 1 = sequence parallelism off
    vpp: int = 0  # NEXT-4: virtual pipeline stages per GPU (interleaved 1F1B); 0/1 = off
    wb: int = 0  # NEXT-4: bytes per parameter of weights / gradients / optimizer states (0 = 2 / 4 / 12)
    gb: int = 0
    ob: int = 0
    name: str = ""
    caps_bytes: Optional[List[int]] = None  # capacities given in bytes (overrides caps_gb)

    @property
    def cap_bytes(self) -> List[int]:
        if self.caps_bytes is not None:
            return list(self.caps_bytes)
        return [g * GIB for g in self.caps_gb]

    def with_models(self, models) -> "Space":
        return dataclasses.replace(self, models=list(models))


SEQ6 = [4096 << i for i in range(6)]  # 4K .. 128K


def c4_models() -> List[Tuple[int, int, int, int, int, int]]:
    """Synthetic Llama-shape grid (BASELINE.json configs[3]):
    h = 1024..16384 step 128 with head dim 128 (a = h/128); k in {1,2,4,8,16,a}
    that divide a; h_ffn = roundup(m h, 256) for m in {8/3, 7/2, 4};
    L = 16..128 step 4; v in 8 vocabularies.  Order: h, k, m, L, v ascending."""
    vocabs = [32000, 32768, 50304, 65536, 100352, 128256, 152064, 256000]
    out = []
    for h in range(1024, 16384 + 1, 128):
        a = h // 128
        ks = sorted({k for k in (1, 2, 4, 8, 16, a) if a % k == 0})
        for k in ks:
            for num, den in ((8, 3), (7, 2), (4, 1)):
                f = -(-(num * h) // (den * 256)) * 256
                for L in range(16, 128 + 1, 4):
                    for v in vocabs:
                        out.append((h, f, L, a, k, v))
    return out


def config(name: str, **kw) -> Space:
    """The BASELINE.json configs as concrete spaces.

    C1  configs[0]  Llama-2-7B on 8 GPUs, b in {1,2,4}, s = 4096 (240 configs)
    C3  configs[2]  Llama-3-70B on 1024 GPUs, b 1..16, s 4K..128K, rc, do
    C4  configs[3]  synthetic grid on 4096 GPUs (~7.7e9 configs)
    C5  configs[4]  C4 grid x N = 8..16384 (powers of two), uneven PP allowed
    (C2, the paper's 454 cells, is a list: see paper_cells())."""
    if name == "C1":
        sp = Space(models=[PRESETS["llama2-7b"]], world=[8], caps_gb=[94, 192], mbs=[1, 2, 4],
                   seq=[4096], name="C1")
    elif name == "C3":
        sp = Space(models=[PRESETS["llama3-70b"]], world=[1024], caps_gb=[40, 80, 94, 192],
                   mbs=list(range(1, 17)), seq=SEQ6, name="C3")
    elif name == "C4":
        sp = Space(models=c4_models(), world=[4096], caps_gb=[40, 80, 94, 192],
                   mbs=list(range(1, 17)), seq=SEQ6, name="C4")
    elif name == "C5":
        sp = Space(models=c4_models(), world=[8 << i for i in range(12)],
                   caps_gb=[40, 80, 94, 192], mbs=list(range(1, 17)), seq=SEQ6, uneven=1,
                   name="C5")
    else:
        raise KeyError(name)
    return dataclasses.replace(sp, **kw) if kw else sp


def load_paper_tables() -> List[dict]:
    """The ten transcribed tables (tests/golden/paper_tables.csv, one row per
    printed cell, with the PAPER.md line it comes from)."""
    with (GOLDEN / "paper_tables.csv").open() as fh:
        rows = list(csv.DictReader(fh))
    for r in rows:
        for k in ("gpu_gb", "seq", "tp", "cp", "pp", "mbs", "n_gpus", "line"):
            r[k] = int(r[k])
    return rows


def paper_cells() -> List[dict]:
    """C2 (BASELINE.json configs[1]): the 454 estimate cells as explicit configs.
    GBS is 1,024 in every experiment; d = N / (t c p)."""
    out = []
    for r in load_paper_tables():
        if r["kind"] != "est":
            continue
        N, t, c, p = r["n_gpus"], r["tp"], r["cp"], r["pp"]
        out.append(dict(r, model_shape=PRESETS[r["model"]], d=N // (t * c * p), gbs=1024))
    return out


def random_models(n: int, seed: int = 241106465, small: bool = False):
    """Seeded random Llama-like shapes satisfying k | a | h."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        if small:
            hd = int(rng.choice([2, 4, 8]))
            a = int(rng.choice([1, 2, 4, 6, 8]))
        else:
            hd = int(rng.choice([64, 80, 96, 128, 256]))
            a = int(rng.choice([8, 12, 16, 24, 32, 40, 48, 64, 96, 128]))
        h = hd * a
        k = int(rng.choice([d for d in range(1, a + 1) if a % d == 0]))
        f = int(rng.integers(1, 9)) * h // 2 if small else int(rng.integers(2, 33)) * 256
        L = int(rng.integers(1, 17)) if small else int(rng.integers(1, 161))
        v = int(rng.integers(2, 65)) * (8 if small else 1000)
        if f <= 0:
            continue
        out.append((h, f, L, a, k, v))
    return out


def random_world_sizes(seed: int, n: int = 4) -> List[int]:
    """Includes non-power-of-two world sizes (exercise the ceil reading R8)."""
    rng = np.random.default_rng(seed)
    base = [8, 12, 24, 48, 96, 6, 10, 18, 64, 128, 40, 72]
    return sorted(set(int(x) for x in rng.choice(base, size=n, replace=False)))
