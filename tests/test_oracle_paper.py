"""Pin the oracle to the numbers the paper prints (CPU only).

Fixtures: tests/golden/paper_tables.csv (every cell of the ten result tables,
transcribed by tests/golden/extract_paper_tables.py with its PAPER.md line) and
tests/golden/errata.csv (the ten cells the canonical reading does not print
identically, each with the evidence that the paper, not the oracle, is off).
"""
import csv
from fractions import Fraction

import pytest

import me_inputs as mi

GIB = 1 << 30


def round_half_up(x: Fraction, nd: int) -> Fraction:
    q = Fraction(1, 10 ** nd)
    return Fraction((x / q + Fraction(1, 2)).__floor__()) * q


def truncate(x: Fraction, nd: int) -> Fraction:
    q = Fraction(1, 10 ** nd)
    return Fraction((x / q).__floor__()) * q


def decimals(txt: str) -> int:
    return len(txt.split(".")[1]) if "." in txt else 0


def cell_total(oracle_mod, r, n_gpus=None):
    N = n_gpus or r["n_gpus"]
    t, c, p = r["tp"], r["cp"], r["pp"]
    e = oracle_mod.estimate(mi.PRESETS[r["model"]], d=N // (t * c * p), t=t, p=p, c=c,
                            b=r["mbs"], s=r["seq"])
    return e["total"]


def load_errata():
    with (mi.GOLDEN / "errata.csv").open() as fh:
        rows = list(csv.DictReader(fh))
    return {(r["table"], int(r["tp"]), int(r["cp"]), int(r["pp"]), int(r["mbs"]),
             int(r["n_gpus"])): r for r in rows}


def key(r):
    return (r["table"], r["tp"], r["cp"], r["pp"], r["mbs"], r["n_gpus"])


def test_fixture_shape():
    rows = mi.load_paper_tables()
    est = [r for r in rows if r["kind"] == "est"]
    thr = [r for r in rows if r["kind"] == "thr"]
    # "454 experiments" = the non-dash cells of the five measured tables
    assert len(est) == 454 and len(thr) == 454
    assert {key(r)[1:] + (r["model"], r["seq"], r["gpu_gb"]) for r in est} == \
           {key(r)[1:] + (r["model"], r["seq"], r["gpu_gb"]) for r in thr}
    # "-" cells are exactly the ones with t*c*p > N
    for r in est:
        assert r["tp"] * r["cp"] * r["pp"] <= r["n_gpus"]
        assert r["n_gpus"] % (r["tp"] * r["cp"] * r["pp"]) == 0
        # GBS 1,024 splits evenly and m >= p in every cell (R17)
        d = r["n_gpus"] // (r["tp"] * r["cp"] * r["pp"])
        assert 1024 % (d * r["mbs"]) == 0 and 1024 // (d * r["mbs"]) >= r["pp"]


def test_454_estimate_cells(oracle_mod):
    """444 cells print R* bytes / 2^30 rounded half-up at the printed decimals;
    the other 10 are the listed errata (5 truncations, 5 typos)."""
    errata = load_errata()
    exact = 0
    for r in mi.paper_cells():
        g = Fraction(cell_total(oracle_mod, r), GIB)
        printed = Fraction(r["text"])
        nd = decimals(r["text"])
        if key(r) in errata:
            assert round_half_up(g, nd) != printed, key(r)
            continue
        assert round_half_up(g, nd) == printed, (key(r), float(g), r["text"], r["line"])
        exact += 1
    assert exact == 444


def test_errata_evidence(oracle_mod):
    """Each erratum is shown to be the paper's slip, not an oracle mismatch."""
    cells = {key(r): r for r in mi.paper_cells()}
    for k, e in load_errata().items():
        r = cells[k]
        g = Fraction(cell_total(oracle_mod, r), GIB)
        printed = Fraction(e["printed"])
        nd = decimals(e["printed"])
        if e["kind"] == "truncated":
            assert truncate(g, nd) == printed
        elif e["kind"] == "row_shift":
            # P:701 prints, at N GPUs, what R* gives at 2N GPUs
            g2 = Fraction(cell_total(oracle_mod, r, n_gpus=2 * r["n_gpus"]), GIB)
            assert round_half_up(g2, nd) == printed
        elif e["kind"] == "copy_typo":
            # another printed cell with identical R* bytes prints the rounded value
            tot = cell_total(oracle_mod, r)
            twins = [o for kk, o in cells.items() if kk != k and cell_total(oracle_mod, o) == tot]
            assert twins and all(Fraction(o["text"]) == round_half_up(g, nd) for o in twins)
            assert abs(printed - round_half_up(g, nd)) == 1
        elif e["kind"] == "digit_typo":
            a, b = e["printed"], f"{float(round_half_up(g, nd)):.{nd}f}"
            assert len(a) == len(b) and sum(x != y for x, y in zip(a, b)) == 1
        else:
            raise AssertionError(e)


def test_454_colours(oracle_mod):
    """Colour = green (<= 80% of capacity), yellow (<= 100%), red (> 100%), with
    capacities 40 / 94 read as GiB (reading R2); ties inclusive (R3)."""
    for r in mi.paper_cells():
        tot = cell_total(oracle_mod, r)
        cap = r["gpu_gb"] * GIB
        col = "green" if tot * 5 <= cap * 4 else ("yellow" if tot <= cap else "red")
        assert col == r["colour"], key(r)
        assert oracle_mod.cap_mask(tot, [cap]) == (1 if col == "green" else 0)


def test_measured_tables_colours_match_estimates(oracle_mod):
    """The measured tables use the same colours as the estimate tables, and the
    80% rule holds on every measured run: no cell estimated <= 80% went OOM
    (P:27)."""
    est = {key(r)[1:] + (r["model"], r["seq"], r["gpu_gb"]): r for r in mi.paper_cells()}
    confusion = {}
    for r in mi.load_paper_tables():
        if r["kind"] != "thr":
            continue
        e = est[key(r)[1:] + (r["model"], r["seq"], r["gpu_gb"])]
        assert r["colour"] == e["colour"], key(r)
        tot = cell_total(oracle_mod, e)
        green = tot * 5 <= r["gpu_gb"] * GIB * 4
        oom = r["text"] == "OOM"
        if green:
            assert not oom, key(r)
        confusion[(e["colour"], oom)] = confusion.get((e["colour"], oom), 0) + 1
    assert confusion == {("green", False): 207, ("yellow", False): 34, ("yellow", True): 42,
                         ("red", True): 171}


@pytest.mark.parametrize("model,N,t,c,p,b,s,gib", [
    # in-text anchors
    ("llama3.1-8b", 4, 1, 2, 1, 1, 8192, "89.95"),
    ("llama3.1-8b", 4, 2, 1, 1, 1, 8192, "67.52"),
    ("llama3.1-8b", 8, 4, 1, 2, 1, 8192, "27.2"),
    ("llama3.1-70b", 64, 8, 1, 8, 1, 8192, "45.95"),
])
def test_in_text_anchors(oracle_mod, model, N, t, c, p, b, s, gib):
    e = oracle_mod.estimate(mi.PRESETS[model], d=N // (t * c * p), t=t, p=p, c=c, b=b, s=s)
    assert round_half_up(Fraction(e["total"], GIB), decimals(gib)) == Fraction(gib)


def test_alternative_readings_fail(oracle_mod):
    """The readings the tables pin: each alternative fails many
    cells, so a plausible slip in the oracle would be caught above."""
    cells = mi.paper_cells()

    def n_fail(fn):
        bad = 0
        for r in cells:
            printed = Fraction(r["text"])
            nd = decimals(r["text"])
            g = fn(r)
            if round_half_up(g, nd) != printed and truncate(g, nd) != printed:
                bad += 1
        return bad

    def base(r):
        return oracle_mod.estimate(mi.PRESETS[r["model"]], d=r["d"], t=r["tp"], p=r["pp"],
                                   c=r["cp"], b=r["mbs"], s=r["seq"])

    # GB read as 1e9 bytes instead of GiB (R1)
    assert n_fail(lambda r: Fraction(base(r)["total"], 10 ** 9)) >= 440
    # optimizer sharded over d only (not d*c, R7)
    def opt_d_only(r):
        e = base(r)
        return Fraction(e["total"] - e["optim"] + e["optim"] * r["cp"], GIB)
    assert n_fail(opt_d_only) >= 250
    # activations not divided by c (R12)
    def act_no_c(r):
        e = base(r)
        act = e["act_layers"] + e["act_embed"] + e["act_head"]
        return Fraction(e["total"] + act * (r["cp"] - 1), GIB)
    assert n_fail(act_no_c) >= 250
