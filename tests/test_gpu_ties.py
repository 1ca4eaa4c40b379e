"""The 80% rule at its boundary, through every kernel path.

P:420: a configuration is feasible when its estimate is "at or below 80%" of
the capacity; reading R3 makes the tie inclusive: total <= floor(cap * 4/5).
The GPU takes this decision in several strength-reduced forms (the survivor
bound umax of a row, the binary searches of the row counts, the carry-chain
masks of the output kernels, the global-batch path that evaluates every
total, the NEXT-1 two-stage bound, me_estimate_batch's compare), so each is
driven with capacities whose threshold equals a configuration's total exactly
and is one byte below it, and compared with the oracle (exact 128-bit
compare total * den <= cap * num)."""
import dataclasses

import numpy as np
import pytest

import me_inputs as mi

pytestmark = pytest.mark.gpu

MODES = (0, 1, 2, 3)  # COUNT, INDEX, FULL, RECORDS


@pytest.fixture(scope="module")
def me():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2411_06465_b200 as me
    torch.cuda.set_device(0)
    return me


def tie_caps(total):
    """capacities whose 4/5 threshold is exactly total, and total - 1"""
    eq = -(-5 * total // 4)
    lo = -(-5 * (total - 1) // 4)
    assert eq * 4 // 5 == total and lo * 4 // 5 == total - 1
    return eq, lo


def compare(me, oracle_mod, sp, env=None):
    plan = me.Plan(sp)
    idx, rows, n, caps = oracle_mod.sweep(sp, threads=8)
    for mode in MODES:
        res = plan.sweep(mode=mode)
        assert res.status() == 0
        assert res.counts()[0] == n, mode
        assert res.cap_counts() == caps, mode
        if mode:
            got = res.to_host()
            assert np.array_equal(got["index_mask"], idx), mode
            if mode >= 2:
                assert np.array_equal(got["total"], rows[:, 6])
    return idx, rows


SPACES = {
    "paper": dict(),                                  # umax path, binary-search counts
    "gbs": dict(gbs=1024),                            # every total evaluated (R17)
    "stage_max": dict(stage_max=1, uneven=1),         # two-stage bound (NEXT-1)
    "stage_max_gbs": dict(stage_max=1, uneven=1, gbs=512),
}


@pytest.mark.parametrize("sparse", ["2", "0"], ids=["two-phase", "positional"])
@pytest.mark.parametrize("kind", list(SPACES))
def test_exact_tie_every_path(me, oracle_mod, monkeypatch, kind, sparse):
    monkeypatch.setenv("ME_SPARSE", sparse)
    kw = SPACES[kind]
    base = mi.Space(models=[mi.PRESETS["llama3.1-8b"], mi.PRESETS["llama2-13b"]], world=[16, 64],
                    caps_gb=[80], mbs=[1, 2, 4], seq=[4096, 8192], **kw)
    # totals of a few configurations of the space, from the oracle
    idx, rows, n, _ = oracle_mod.sweep(dataclasses.replace(base, caps_gb=[1 << 20]), threads=8)
    rng = np.random.default_rng(3)
    for k in rng.choice(len(idx), size=4, replace=False):
        T = int(rows[k, 6])
        eq, lo = tie_caps(T)
        # capacities in bytes: both orders, and each alone (then it is the
        # largest threshold, i.e. the survivor bound)
        for caps in ([eq, lo], [lo, eq], [eq], [lo]):
            oi, orows = compare(me, oracle_mod, dataclasses.replace(base, caps_bytes=caps))
            at = np.nonzero((oi & np.uint64((1 << 56) - 1)) == idx[k] & np.uint64((1 << 56) - 1))[0]
            if caps == [lo]:
                assert len(at) == 0  # one byte over: infeasible
            else:
                assert len(at) == 1
                mask = int(oi[at[0]] >> np.uint64(56))
                assert mask & (1 << caps.index(eq))
                if lo in caps:
                    assert not mask & (1 << caps.index(lo))


def test_exact_tie_estimate_batch(me, oracle_mod):
    shape = mi.PRESETS["llama3.1-70b"]
    cfgs = [dict(d=2, t=8, p=4, c=2, b=1, s=8192), dict(d=1, t=4, p=8, c=1, b=2, s=4096, rc=1),
            dict(d=3, t=2, p=1, c=1, b=1, s=4096, dopt=0), dict(d=8, t=8, p=2, c=4, b=4, s=32768, gbs=64)]
    for cfg in cfgs:
        T = oracle_mod.estimate(shape, **cfg)["total"]
        eq, lo = tie_caps(T)
        rows, mask, status = me.me_estimate_batch([shape], None, [cfg], caps_bytes=[eq, lo])
        assert status[0] == 0 and int(rows[0, 6]) == T
        assert mask[0] == 1 == oracle_mod.cap_mask(T, [eq, lo])


def test_threshold_clamp_huge_capacities(me, oracle_mod):
    """cap * num / den >= 2^64 (num/den up to 1024): the threshold must not wrap"""
    caps = [(1 << 64) - 1, 1 << 62, 40 << 30]
    for num, den in ((1024, 1), (4, 5), (1024, 3)):
        sp = mi.Space(models=[mi.PRESETS["llama3.1-8b"]], world=[8, 64], caps_gb=[], mbs=[1, 2],
                      seq=[4096, 131072], thr_num=num, thr_den=den, uneven=1, caps_bytes=caps)
        compare(me, oracle_mod, sp)
    rows, mask, status = me.me_estimate_batch([mi.PRESETS["llama3.1-8b"]], None,
                                              [dict(d=1, t=1, p=1, c=1, b=1, s=4096)], caps_bytes=caps, thr=(1024, 1))
    assert status[0] == 0 and mask[0] == 0b111


def test_domain_limits(me, oracle_mod):
    """the exact-u64 domain of a sweep (me.h me_plan_create): its largest
    values are accepted and evaluated exactly; one past is ME_EINVAL"""
    big = (32768, 131072, 256, 256, 256, 524288)
    sp = mi.Space(models=[big], world=[1 << 20], caps_gb=[1 << 20, 192], mbs=[1, 64], seq=[1 << 20],
                  max_t=4, max_c=4, max_p=4)
    compare(me, oracle_mod, sp)
    for bad in [(65536, 131072, 256, 256, 256, 524288), (32768, 131072 * 2, 256, 256, 256, 524288),
                (32768, 131072, 512, 256, 256, 524288), (32768, 131072, 256, 256, 256, 524288 * 2)]:
        with pytest.raises(me.MEError) as e:
            me.Plan(mi.Space(models=[bad], world=[8], caps_gb=[80], mbs=[1], seq=[4096]))
        assert e.value.status == me._abi.ME_EINVAL
    for kw in (dict(mbs=[65]), dict(seq=[(1 << 20) + 1]), dict(world=[(1 << 20) + 1])):
        args = dict(models=[mi.PRESETS["llama3.1-8b"]], world=[8], caps_gb=[80], mbs=[1], seq=[4096])
        args.update(kw)
        with pytest.raises(me.MEError) as e:
            me.Plan(mi.Space(**args))
        assert e.value.status == me._abi.ME_EINVAL
