"""NEXT-3 (safety-rule validation) and NEXT-2 (colouring) on the GPU path."""
import numpy as np
import pytest

import me_inputs as mi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def me():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2411_06465_b200 import build
    build.build()
    import paper_2411_06465_b200 as me
    return me


def measured_runs():
    """The paper's 454 measured outcomes."""
    out = []
    for r in mi.load_paper_tables():
        if r["kind"] != "thr":
            continue
        N, t, c, p = r["n_gpus"], r["tp"], r["cp"], r["pp"]
        out.append(dict(model_shape=mi.PRESETS[r["model"]], d=N // (t * c * p), t=t, p=p, c=c, b=r["mbs"],
                        s=r["seq"], gbs=1024, cap_gb=r["gpu_gb"], oom=r["text"] == "OOM", paper_colour=r["colour"],
                        line=r["line"]))
    return out


def test_safety_rule_confusion(me, oracle_mod):
    from paper_2411_06465_b200 import validate
    runs = measured_runs()
    cl = validate.classify(runs)
    assert all(r["colour"] == r["paper_colour"] for r in cl)
    for r in cl[::37]:
        e = oracle_mod.estimate(r["model_shape"], d=r["d"], t=r["t"], p=r["p"], c=r["c"], b=r["b"], s=r["s"],
                                gbs=1024)
        assert e["total"] == r["total"]
    assert validate.confusion(cl) == {("green", False): 207, ("yellow", False): 34, ("yellow", True): 42,
                                      ("red", True): 171}
    rep = validate.report(runs)
    assert rep["rule_holds"] and rep["green_oom"] == 0 and rep["red_trained"] == 0


def three_class(sp, C):
    """the space swept with capacities {C, 5C/4, UINT64_MAX} under the 4/5 rule:
    bit 0 = green (<= 80% of C), bit 1 = green or yellow (<= C), bit 2 = any
    (red included); 4 | C makes 5C/4 * 4/5 = C exact"""
    import dataclasses
    assert C % 4 == 0
    return dataclasses.replace(sp, caps_gb=[], caps_bytes=[C, 5 * C // 4, (1 << 64) - 1], thr_num=4, thr_den=5)


@pytest.mark.parametrize("name", ["C1", "C3", "rand", "a100"])
@pytest.mark.parametrize("mode", [1, 2, 3], ids=["index", "full", "records"])
def test_rank_matches_oracle(me, oracle_mod, name, mode):
    """me_result_rank's top-k per segment (survey key, classes from the masks)
    equals oracle.rank's (classes from the exact totals, plain tuple sort)."""
    gpn = 4
    if name == "rand":
        sp = mi.Space(models=mi.random_models(4, seed=41), world=[16, 24, 64], caps_gb=[], mbs=[1, 2, 4],
                      seq=[4096, 8192], uneven=1)
        C = 24 << 30
    elif name == "a100":
        sp = mi.Space(models=[mi.PRESETS["llama3.1-8b"]], world=[8, 16, 32, 64, 128, 256], caps_gb=[],
                      mbs=[1, 2, 4, 8], seq=[8192], gbs=1024, rc_mask=1, do_mask=2)
        C, gpn = 40 << 30, 8
    else:
        sp = mi.config(name)
        C = 80 << 30
    k = 5
    res = me.Plan(three_class(sp, C)).sweep(mode=mode)
    got = res.rank(green_cap=0, yellow_cap=1, gpus_per_node=gpn, k=k)
    ref = oracle_mod.rank(sp, C, gpus_per_node=gpn, k=k)
    n_seg = len(sp.models) * len(sp.world)
    for seg in range(n_seg):
        g = [(r["index"], r["cls"], (r["t"], r["c"], r["p"], r["b"])) for r in got[seg]]
        assert g == ref.get(seg, []), (name, seg)
        for r in got[seg]:
            if sp.gbs:
                assert r["microbatches"] == sp.gbs // (r["d"] * r["b"])
                assert r["bubble"] == (r["p"] - 1, r["microbatches"])


def test_rank_picks_paper_choice(me):
    """Llama-3.1-8B, s = 8192, A100 40 GB, GBS 1,024: at 16 GPUs the
    top green row is (4, 1, 1, 1) (bold 194.97); at 256 GPUs
    the paper's optimum (4, 1, 1, 2) is yellow and ranks first once
    the yellow class counts as feasible (yellow_cap as the green slot), the
    best green one being (4, 1, 1, 1).  (2, 1, 2, 1) has 128 microbatches on 32
    GPUs and 16 on 256: the bubble grows 8x."""
    sp = mi.Space(models=[mi.PRESETS["llama3.1-8b"]], world=[16, 32, 256], caps_gb=[], mbs=[1, 2, 4, 8],
                  seq=[8192], gbs=1024, rc_mask=1, do_mask=2, max_t=8)
    res = me.Plan(three_class(sp, 40 << 30)).sweep(mode=me.ME_OUT_INDEX)
    top = res.rank(green_cap=0, yellow_cap=1, gpus_per_node=8, k=1)
    assert [(r[0]["t"], r[0]["c"], r[0]["p"], r[0]["b"], r[0]["cls"]) for r in top] == [(4, 1, 1, 1, 0)] * 3
    top100 = res.rank(green_cap=1, gpus_per_node=8, k=1)
    assert (top100[2][0]["t"], top100[2][0]["c"], top100[2][0]["p"], top100[2][0]["b"]) == (4, 1, 1, 2)
    allrows = res.rank(green_cap=0, yellow_cap=1, gpus_per_node=8, k=10000)
    bub = {}
    for seg, N in enumerate(sp.world):
        for r in allrows[seg]:
            if (r["t"], r["c"], r["p"], r["b"]) == (2, 1, 2, 1):
                bub[N] = r["bubble"]
    assert bub[32] == (1, 128) and bub[256] == (1, 16)


def test_three_class_colouring_with_red(me, oracle_mod):
    """all three classes of a sweep from the masks (capacities C, 5C/4 and
    UINT64_MAX under 4/5): every configuration is in the result, red ones
    with bit 2 only; compared with the exact totals"""
    C = 40 << 30
    sp = mi.Space(models=[mi.PRESETS["llama3.1-8b"], mi.PRESETS["llama2-13b"]], world=[64, 256], caps_gb=[],
                  mbs=[1, 2, 4, 8], seq=[4096, 8192, 16384], gbs=1024)
    sp3 = three_class(sp, C)
    res = me.Plan(sp3).sweep(mode=me.ME_OUT_RECORDS)
    got = res.to_host()
    assert res.counts()[0] == oracle_mod.space_size(sp)
    mask = got["index_mask"] >> np.uint64(56)
    cls = np.where(mask & np.uint64(1), 0, np.where(mask & np.uint64(2), 1, 2))
    ref = np.array([oracle_mod.feasibility_class(int(t), C) for t in got["total"]])
    assert np.array_equal(cls, ref) and set(ref.tolist()) == {0, 1, 2}
    idx, rows, n, caps = oracle_mod.sweep(sp3)
    assert np.array_equal(got["index_mask"], idx)


def test_three_class_colouring_sweep(me, oracle_mod):
    """NEXT-2 3-class colouring of a sweep (green <= 80 %, yellow <= 100 %,
    red > 100 % of C; caption P:420): capacities {C, 5C/4} at the 4/5 rule
    give bit 0 = green and bit 1 = green or yellow, exactly (5C/4 * 4/5 = C
    for C a multiple of 4 bytes).  Checked row by row against the totals."""
    C = 40 << 30
    sp = mi.Space(models=[mi.PRESETS["llama3.1-8b"], mi.PRESETS["llama2-13b"]], world=[64, 256],
                  caps_gb=[40, 50], mbs=[1, 2, 4, 8], seq=[4096, 8192, 16384], gbs=1024)
    res = me.Plan(sp).sweep(mode=me.ME_OUT_RECORDS)
    got = res.to_host()
    mask = got["index_mask"] >> np.uint64(56)
    total = got["total"]
    assert len(total) > 0
    green = total * np.uint64(5) <= np.uint64(C * 4)
    yellow_or_green = total <= np.uint64(C)
    assert np.array_equal((mask & np.uint64(1)) == 1, green)
    assert np.array_equal((mask >> np.uint64(1) & np.uint64(1)) == 1, yellow_or_green)
    # the survivors are exactly the oracle's (any bit set: total <= C)
    idx, rows, n, caps = oracle_mod.sweep(sp)
    assert np.array_equal(got["index_mask"], idx)
    assert caps[0] == int(green.sum()) and caps[1] == n
