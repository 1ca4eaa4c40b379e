"""NEXT-3: validation of the 80% safety rule against measured training runs.

The paper's claim: a configuration whose
estimate is at most 80% of the GPU memory never ran out of memory in its 454
experiments.  Given measured runs (configuration, capacity, OOM or not), this
module classifies every run with the estimator on the GPU (me_estimate_batch)
as green (<= 80% of capacity), yellow (<= 100%) or red (> 100%) -- the colours
of the paper's tables (caption) -- and reports the confusion matrix and
the anomalies: green runs that went OOM (rule violations) and red runs that
trained (estimator over-estimates).  Capacities are GiB (reading R2).
"""
from __future__ import annotations

from typing import Dict, Iterable, List, Sequence, Tuple

import numpy as np

GIB = 1 << 30


def classify(runs: Sequence[dict]) -> List[dict]:
    """runs: dicts with model_shape (h, h_ffn, L, a, k, v), d, t, p, c, b, s,
    optional gbs, cap_gb.  Returns the runs with total (bytes) and colour.
    The colours are the GPU's capacity masks (me_estimate_batch): bit j at the
    4/5 rule = green for capacity j, at 1/1 = within capacity j."""
    from . import me_estimate_batch

    shapes: List[Tuple[int, ...]] = []
    index: Dict[Tuple[int, ...], int] = {}
    ids, cfgs, slot = [], [], []
    caps = sorted({int(r["cap_gb"]) for r in runs})
    cap_bytes = [c * GIB for c in caps]
    for r in runs:
        key = tuple(r["model_shape"])
        if key not in index:
            index[key] = len(shapes)
            shapes.append(key)
        ids.append(index[key])
        cfgs.append(dict(d=r["d"], t=r["t"], p=r["p"], c=r["c"], b=r["b"], s=r["s"], gbs=r.get("gbs", 0)))
        slot.append(caps.index(int(r["cap_gb"])))
    rows, m80, status = me_estimate_batch(shapes, ids, cfgs, caps_bytes=cap_bytes, thr=(4, 5))
    if status.any():
        bad = int(np.flatnonzero(status)[0])
        raise ValueError(f"run {bad}: estimator precondition failed (status {int(status[bad])})")
    _, m100, _ = me_estimate_batch(shapes, ids, cfgs, caps_bytes=cap_bytes, thr=(1, 1))
    totals = [int(t) for t in rows[:, 6]]
    green = [bool(m80[i] >> q & 1) for i, q in enumerate(slot)]
    within = [bool(m100[i] >> q & 1) for i, q in enumerate(slot)]
    out = []
    for r, tot, g, w in zip(runs, totals, green, within):
        colour = "green" if g else ("yellow" if w else "red")
        out.append(dict(r, total=int(tot), colour=colour))
    return out


def confusion(classified: Iterable[dict]) -> Dict[Tuple[str, bool], int]:
    """(colour, went OOM) -> number of runs."""
    out: Dict[Tuple[str, bool], int] = {}
    for r in classified:
        k = (r["colour"], bool(r["oom"]))
        out[k] = out.get(k, 0) + 1
    return out


def anomalies(classified: Iterable[dict]) -> Dict[str, List[dict]]:
    """Green runs that went OOM violate the 80% rule; red runs that trained
    show the estimate above the real footprint."""
    cl = list(classified)
    return {"green_oom": [r for r in cl if r["colour"] == "green" and r["oom"]],
            "red_trained": [r for r in cl if r["colour"] == "red" and not r["oom"]]}


def report(runs: Sequence[dict]) -> dict:
    cl = classify(runs)
    conf = confusion(cl)
    an = anomalies(cl)
    return {"runs": len(cl), "confusion": {f"{c}/{'oom' if o else 'ok'}": n for (c, o), n in sorted(conf.items())},
            "rule_holds": not an["green_oom"], "green_oom": len(an["green_oom"]),
            "red_trained": len(an["red_trained"])}
