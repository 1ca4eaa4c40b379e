"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bit-exact on every record: flat index, capacity mask, six terms and total
(all integers; there is no tolerance).  Small spaces are compared in full;
the BASELINE.json full-size spaces (C4, C5) on sampled windows in the same
launch configuration bench.py uses, plus properties that hold at any size."""
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
    torch.cuda.set_device(0)
    return me


def oracle_rows(oracle_mod, sp, begin=0, end=0, threads=8):
    idx, rows, n, caps = oracle_mod.sweep(sp, begin, end, threads=threads)
    return idx, rows, n, caps


def assert_same(me, res, idx, rows, n, caps, mode):
    lo, gl, off = res.counts()
    assert lo == n and gl == n and off == 0
    assert res.cap_counts() == caps
    if mode == me.ME_OUT_COUNT:
        return
    got = res.to_host()
    assert np.array_equal(got["index_mask"], idx)
    if mode in (me.ME_OUT_FULL, me.ME_OUT_RECORDS):
        for j, k in enumerate(me.TERMS):
            assert np.array_equal(got[k], rows[:, j]), k


# ---------------------------------------------------------------- single estimates
def test_estimate_454_paper_cells(me, oracle_mod):
    """C2 (BASELINE.json configs[1]): the paper's 454 cells through me_estimate_batch."""
    cells = mi.paper_cells()
    shapes = [mi.PRESETS["llama3.1-8b"], mi.PRESETS["llama3.1-70b"]]
    ids = [0 if c["model"] == "llama3.1-8b" else 1 for c in cells]
    for gbs in (0, 1024):
        cfgs = [dict(d=c["d"], t=c["tp"], p=c["pp"], c=c["cp"], b=c["mbs"], s=c["seq"], gbs=gbs) for c in cells]
        for cap in (40, 94):
            rows, mask, status = me.me_estimate_batch(shapes, ids, cfgs, caps_bytes=[cap << 30])
            assert not status.any()
            for i, c in enumerate(cells):
                e = oracle_mod.estimate(shapes[ids[i]], **cfgs[i])
                assert rows[i].tolist() == [e[k] for k in oracle_mod.TERMS]
                assert mask[i] == oracle_mod.cap_mask(e["total"], [cap << 30])
    # the colour of the table the cell comes from (80% -> green)
    rows, mask, _ = me.me_estimate_batch(shapes, ids, [dict(d=c["d"], t=c["tp"], p=c["pp"], c=c["cp"], b=c["mbs"],
                                                            s=c["seq"]) for c in cells],
                                         caps_bytes=[40 << 30, 94 << 30])
    for i, c in enumerate(cells):
        bit = 0 if c["gpu_gb"] == 40 else 1
        assert bool(mask[i] >> bit & 1) == (c["colour"] == "green")


def random_cfgs(rng, shape, n):
    h, f, L, a, k, v = shape
    out = []
    for _ in range(n):
        t = int(rng.choice([1, 2, 3, 4, 8, 16]))
        c = int(rng.choice([1, 2, 3, 4, 8]))
        p = int(rng.choice([1, 2, 3, 4, 5, 8, L, L + 1]))
        d = int(rng.integers(1, 40))
        b = int(rng.choice([1, 2, 3, 4, 16]))
        s = int(rng.choice([1024, 3072, 4096, 8192, 12288]))
        cfg = dict(d=d, t=t, p=p, c=c, b=b, s=s, gbs=int(rng.choice([0, 0, 96, 1024, 1000])),
                   rc=int(rng.integers(0, 2)), dopt=int(rng.integers(0, 2)), uneven=int(rng.integers(0, 2)))
        if rng.random() < 0.2 and p > 1:
            cfg["L0"] = int(rng.integers(1, L + 1))
        out.append(cfg)
    return out


def test_estimate_random_with_status(me, oracle_mod):
    rng = np.random.default_rng(241106465)
    shapes = mi.random_models(24, seed=5) + [mi.PRESETS[k] for k in ("llama2-7b", "llama2-13b", "llama3.1-70b")]
    caps = [40 << 30, 80 << 30, 94 << 30, 192 << 30]
    for si, shape in enumerate(shapes):
        cfgs = random_cfgs(rng, shape, 200)
        rows, mask, status = me.me_estimate_batch([shape], None, cfgs, caps_bytes=caps)
        for i, cfg in enumerate(cfgs):
            st = oracle_mod.estimate_status(shape, **cfg)
            assert status[i] == st, (shape, cfg)
            if st == 0:
                e = oracle_mod.estimate(shape, **cfg)
                assert rows[i].tolist() == [e[k] for k in oracle_mod.TERMS], (shape, cfg)
                assert mask[i] == oracle_mod.cap_mask(e["total"], caps)


def test_estimate_edge_cases(me, oracle_mod):
    M8 = mi.PRESETS["llama3.1-8b"]
    edge = [
        ((1, 1, 1, 1, 1, 1), dict(d=1, t=1, p=1, c=1, b=1, s=1)),              # unit model
        ((32768, 131072, 256, 256, 256, 524288), dict(d=1, t=1, p=1, c=1, b=64, s=1 << 20)),  # domain max
        ((32768, 131072, 256, 256, 256, 524288), dict(d=1, t=256, p=256, c=1, b=64, s=1 << 20)),
        ((65536, 131072, 4096, 512, 512, 1 << 22), dict(d=1, t=1, p=1, c=1, b=64, s=1 << 24)),  # overflow
        (M8, dict(d=7, t=1, p=1, c=1, b=1, s=8192)),                            # ceil rule, d odd
        (M8, dict(d=1, t=8, p=32, c=1, b=1, s=8192)),                           # p = L
        (M8, dict(d=1, t=8, p=1, c=8192, b=1, s=8192)),                         # c = s
        (M8, dict(d=1, t=1, p=2, c=1, b=4, s=8192, gbs=4)),                     # m = 1 < p
        (M8, dict(d=1, t=1, p=3, c=1, b=1, s=8192, uneven=1)),
        (M8, dict(d=1, t=1, p=3, c=1, b=1, s=8192, L0=30)),
        (M8, dict(d=1, t=1, p=3, c=1, b=1, s=8192, L0=31)),                      # EDIV
        (M8, dict(d=0, t=1, p=1, c=1, b=1, s=8192)),                            # EINVAL
    ]
    for shape, cfg in edge:
        rows, mask, status = me.me_estimate_batch([shape], None, [cfg], caps_bytes=[80 << 30])
        st = oracle_mod.estimate_status(shape, **cfg)
        assert status[0] == st, (shape, cfg)
        if st == 0:
            e = oracle_mod.estimate(shape, **cfg)
            assert rows[0].tolist() == [e[k] for k in oracle_mod.TERMS]
    # me_estimate raises with the oracle's status
    with pytest.raises(me.MEError) as ex:
        me.me_estimate(M8, d=1, t=3, p=1, c=1, b=1, s=8192)
    assert ex.value.status == oracle_mod.EDIV


# ---------------------------------------------------------------- sweeps
def small_spaces():
    yield "C1", mi.config("C1")
    yield "C3", mi.config("C3")
    yield "C3u", mi.config("C3", uneven=1)
    yield "gbs", mi.Space(models=mi.random_models(5, seed=21, small=True), world=[6, 8, 12, 24], caps_gb=[1, 2, 4],
                          mbs=[1, 2, 3], seq=[8, 12, 16, 24], gbs=96, uneven=1, thr_num=9, thr_den=10)
    yield "masks", mi.Space(models=mi.random_models(6, seed=22), world=mi.random_world_sizes(22, 5),
                            caps_gb=[24, 40, 80, 94, 141, 180, 192, 288], mbs=[1, 2, 8], seq=[2048, 4096, 32768],
                            rc_mask=2, do_mask=1, max_t=16, max_p=8)
    yield "one_cap", mi.Space(models=[mi.PRESETS["llama2-70b"], mi.PRESETS["llama2-13b"]], world=[64, 48],
                              caps_gb=[80], mbs=[1, 2], seq=[4096], gpus_per_node=8, rc_mask=1, do_mask=3)


@pytest.mark.parametrize("name,sp", list(small_spaces()), ids=[n for n, _ in small_spaces()])
@pytest.mark.parametrize("mode", [0, 1, 2, 3], ids=["count", "index", "full", "records"])
def test_sweep_small_spaces(me, oracle_mod, name, sp, mode):
    plan = me.Plan(sp)
    assert plan.size == oracle_mod.space_size(sp)
    res = plan.sweep(mode=mode)
    assert res.status() == 0
    assert_same(me, res, *oracle_rows(oracle_mod, sp), mode)


def test_sweep_subranges(me, oracle_mod):
    sp = mi.config("C3", uneven=1)
    plan = me.Plan(sp)
    rng = np.random.default_rng(3)
    ranges = [(0, 1), (5, 5), (31, 33), (1000, 1031), (plan.size - 1, plan.size), (0, 0)]
    ranges += [tuple(sorted(int(x) for x in rng.integers(0, plan.size, 2))) for _ in range(6)]
    for i, (b, e) in enumerate(ranges):
        mode = (me.ME_OUT_FULL, me.ME_OUT_RECORDS)[i & 1]
        res = plan.sweep(b, e, mode=mode)
        if (b, e) == (0, 0):
            e = plan.size
        assert_same(me, res, *oracle_rows(oracle_mod, sp, b, e), mode)


def test_caller_columns_and_overflow(me, oracle_mod):
    import torch
    sp = mi.config("C3")
    plan = me.Plan(sp)
    idx, rows, n, caps = oracle_rows(oracle_mod, sp)
    cols = [torch.full((n + 5,), -1, dtype=torch.int64, device="cuda") for _ in range(8)]
    res = plan.sweep(mode=me.ME_OUT_FULL, out_cols=cols)
    assert res.status() == 0
    assert_same(me, res, idx, rows, n, caps, me.ME_OUT_FULL)
    assert (cols[0][n:] == -1).all()
    rec = torch.full(((n + 3) * 8,), -1, dtype=torch.int64, device="cuda")
    res = plan.sweep(mode=me.ME_OUT_RECORDS, out_cols=[rec])
    assert res.status() == 0
    assert_same(me, res, idx, rows, n, caps, me.ME_OUT_RECORDS)
    assert (rec[n * 8:] == -1).all()
    small_rec = torch.full(((n // 3) * 8 + 8,), -1, dtype=torch.int64, device="cuda")
    res = plan.sweep(mode=me.ME_OUT_RECORDS, out_cols=[small_rec[:(n // 3) * 8]])
    assert res.status() == 7  # ME_ERANGE: rows past the capacity are not written
    assert (small_rec[(n // 3) * 8:] == -1).all()
    got = small_rec[:(n // 3) * 8].view(-1, 8).cpu().numpy().view(np.uint64)
    assert np.array_equal(got[:, 0], idx[: n // 3])
    small = [torch.zeros(n // 2, dtype=torch.int64, device="cuda")]
    res = plan.sweep(mode=me.ME_OUT_INDEX, out_cols=small)
    assert res.status() == 7  # ME_ERANGE
    assert res.counts()[0] == n
    got = small[0].cpu().numpy().view(np.uint64)
    assert np.array_equal(got, idx[: n // 2])


def test_random_model_grid(me, oracle_mod):
    """Seeded random Llama shapes x non-power-of-two world sizes (ceil rule R8)."""
    sp = mi.Space(models=mi.random_models(40, seed=99), world=[24, 96, 120, 1000], caps_gb=[40, 80, 94, 192],
                  mbs=[1, 2, 4], seq=[4096, 8192, 131072], uneven=1)
    plan = me.Plan(sp)
    res = plan.sweep(mode=me.ME_OUT_FULL)
    assert_same(me, res, *oracle_rows(oracle_mod, sp, threads=16), me.ME_OUT_FULL)


@pytest.mark.parametrize("name,mode", [("C4", 2), ("C5", 2), ("C5", 3)], ids=["C4-full", "C5-full", "C5-records"])
def test_full_size_sampled(me, oracle_mod, name, mode):
    """BASELINE.json configs[3]/[4] at full size, in bench.py's launch
    configuration (chunks of bench.CHUNK): windows compared record by record
    with the oracle, sampled rows of whole chunks recomputed one by one, and
    the properties every chunk must have."""
    import torch

    import bench
    sp = mi.config(name)
    plan = me.Plan(sp)
    assert plan.size == oracle_mod.space_size(sp)
    rng = np.random.default_rng(7 if name == "C4" else 8)
    # exact windows (including the first and last indices of the space)
    wins = [(0, 20_000), (plan.size - 20_000, plan.size)]
    wins += [(s, s + 20_000) for s in (int(x) for x in rng.integers(0, plan.size - 20_000, 4))]
    for b, e in wins:
        res = plan.sweep(b, e, mode=mode)
        assert_same(me, res, *oracle_rows(oracle_mod, sp, b, e), mode)
    # whole bench chunks: sampled rows and ordering properties
    chunk = bench.CHUNK
    if mode == me.ME_OUT_RECORDS:
        rec = torch.empty(chunk * 8, dtype=torch.int64, device="cuda")
        out_cols = [rec]
        cols = [rec.view(chunk, 8)[:, j] for j in range(8)]
    else:
        cols = out_cols = [torch.empty(chunk, dtype=torch.int64, device="cuda") for _ in range(8)]
    starts = [0, (plan.size // chunk // 2) * chunk, (plan.size - 1) // chunk * chunk]
    for s in starts:
        e = min(plan.size, s + chunk)
        res = plan.sweep(s, e, mode=mode, out_cols=out_cols)
        assert res.status() == 0
        n = res.counts()[0]
        assert 0 < n <= e - s
        ix = cols[0][:n].cpu().numpy().view(np.uint64)
        index = ix & np.uint64((1 << 56) - 1)
        mask = ix >> np.uint64(56)
        assert (np.diff(index.astype(np.int64)) > 0).all() and index[0] >= s and index[-1] < e
        assert (mask > 0).all() and (mask < 16).all()
        tot = [cols[j][:n].cpu().numpy().view(np.uint64) for j in range(1, 8)]
        assert np.array_equal(tot[0] + tot[1] + tot[2] + tot[3] + tot[4] + tot[5], tot[6])
        assert np.array_equal(tot[1], 2 * tot[0])
        # masks are monotone in capacity: feasible at 40 GiB => feasible at 80, ...
        m = mask.astype(np.int64)
        assert ((m & 1) <= (m >> 1 & 1)).all() and ((m >> 1 & 1) <= (m >> 2 & 1)).all()
        ks = np.sort(rng.choice(n, size=256, replace=False))
        o_rows, o_masks = oracle_mod.points(sp, index[ks])
        for q, k in enumerate(ks):
            assert [int(t[k]) for t in tot] == o_rows[q].tolist(), int(index[k])
            assert int(mask[k]) == int(o_masks[q])


# ---------------------------------------------------------------- NEXT-1: every stage
def test_estimate_stage_matches_oracle(me, oracle_mod):
    rng = np.random.default_rng(17)
    shapes = mi.random_models(12, seed=13) + [mi.PRESETS["llama3.1-8b"], (1024, 2816, 16, 8, 8, 256000)]
    for shape in shapes:
        h, f, L, a, k, v = shape
        for _ in range(25):
            p = int(rng.integers(1, L + 1))
            cfg = dict(d=int(rng.integers(1, 17)), t=1, p=p, c=int(rng.choice([1, 2])), b=int(rng.integers(1, 5)),
                       s=int(rng.choice([4096, 8192])), gbs=int(rng.choice([0, 0, 64, 1024])),
                       rc=int(rng.integers(0, 2)), dopt=int(rng.integers(0, 2)), uneven=1)
            if cfg["gbs"] and cfg["gbs"] % (cfg["d"] * cfg["b"]):
                cfg["gbs"] = 0
            for i in sorted({0, p - 1, int(rng.integers(0, p))}):
                got, which = me.me_estimate_stage(shape, i, **cfg)
                assert which == i
                assert got == oracle_mod.estimate_stage(shape, i, **cfg), (shape, cfg, i)
            got, which = me.me_estimate_stage(shape, me.STAGE_ARGMAX, **cfg)
            ref, arg = oracle_mod.estimate_max(shape, **cfg)
            assert (got, which) == (ref, arg), (shape, cfg)
    with pytest.raises(me.MEError):
        me.me_estimate_stage(mi.PRESETS["llama3.1-8b"], 4, d=1, t=1, p=4, c=1, b=1, s=8192)


@pytest.mark.parametrize("mode", [0, 1, 2, 3], ids=["count", "index", "full", "records"])
@pytest.mark.parametrize("name", ["C3u", "gbs", "rand"])
def test_sweep_stage_max(me, oracle_mod, name, mode):
    """NEXT-1 sweeps: feasibility of the largest pipeline stage."""
    if name == "C3u":
        sp = mi.config("C3", uneven=1, stage_max=1)
    elif name == "gbs":
        sp = mi.Space(models=mi.random_models(5, seed=21, small=True), world=[6, 8, 12, 24], caps_gb=[1, 2, 4],
                      mbs=[1, 2, 3], seq=[8, 12, 16, 24], gbs=96, uneven=1, thr_num=9, thr_den=10, stage_max=1)
    else:
        sp = mi.Space(models=mi.random_models(20, seed=23) + [(1024, 2816, 16, 8, 8, 256000)],
                      world=[8, 24, 64], caps_gb=[24, 40, 80, 192], mbs=[1, 2, 8], seq=[4096, 32768],
                      uneven=1, stage_max=1)
    plan = me.Plan(sp)
    res = plan.sweep(mode=mode)
    assert res.status() == 0
    assert_same(me, res, *oracle_rows(oracle_mod, sp), mode)
    # the first-stage sweep of the same space differs (the last stage binds somewhere)
    if name == "rand":
        import dataclasses
        r0 = me.Plan(dataclasses.replace(sp, stage_max=0)).sweep(mode=me.ME_OUT_COUNT)
        assert r0.counts()[0] != res.counts()[0]


# ---------------------------------------------------------------- NEXT-4: ZeRO stages
def test_estimate_zero_stages(me, oracle_mod):
    rng = np.random.default_rng(29)
    shapes = mi.random_models(10, seed=31) + [mi.PRESETS["llama3.1-70b"]]
    caps = [40 << 30, 80 << 30]
    for shape in shapes:
        cfgs = random_cfgs(rng, shape, 60)
        for cfg in cfgs:
            cfg["zero"] = int(rng.integers(0, 4))
        rows, mask, status = me.me_estimate_batch([shape], None, cfgs, caps_bytes=caps)
        for i, cfg in enumerate(cfgs):
            st = oracle_mod.estimate_status(shape, **cfg)
            assert status[i] == st, (shape, cfg)
            if st == 0:
                e = oracle_mod.estimate(shape, **cfg)
                assert rows[i].tolist() == [e[k] for k in oracle_mod.TERMS], (shape, cfg)
                assert mask[i] == oracle_mod.cap_mask(e["total"], caps)
                if cfg["p"] > 1:
                    for stg in (0, cfg["p"] - 1):
                        got, _ = me.me_estimate_stage(shape, stg, **cfg)
                        assert got == oracle_mod.estimate_stage(shape, stg, **cfg)


@pytest.mark.parametrize("zero", [2, 3])
@pytest.mark.parametrize("stage_max", [0, 1])
def test_sweep_zero_stages(me, oracle_mod, zero, stage_max):
    sp = mi.Space(models=mi.random_models(12, seed=37) + [mi.PRESETS["llama3.1-8b"]], world=[16, 24, 128],
                  caps_gb=[40, 80, 192], mbs=[1, 2, 4], seq=[4096, 16384], uneven=1, zero_stage=zero,
                  stage_max=stage_max)
    res = me.Plan(sp).sweep(mode=me.ME_OUT_FULL)
    assert_same(me, res, *oracle_rows(oracle_mod, sp), me.ME_OUT_FULL)


@pytest.mark.parametrize("env", [{"ME_SERIAL": "1"}, {"ME_SETS": "3"}, {"ME_FUSED_BPS": "1"},
                                 {"ME_SERIAL": "1", "ME_FUSED_BPS": "1"}, {"ME_SPARSE": "0"}, {"ME_SPARSE": "4"},
                                 {"ME_FUSED_MINB": "2"}, {"ME_FUSED_MINB": "3"}, {"ME_K0_FENCE": "0"}],
                         ids=["serial", "sets3", "fused-1bps", "serial-1bps", "positional", "sparse4", "minb2",
                              "minb3", "no-fence"])
def test_pipeline_variants(me, oracle_mod, monkeypatch, env):
    """The launch variants (read at plan creation) give the same rows: serial
    streams, three scratch sets, one fused-kernel block per SM, K3's
    positional row path only (ME_SPARSE=0) or the two-phase path for rows
    with under a quarter survivors."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    spaces = [mi.config("C3", uneven=1),
              mi.Space(models=mi.random_models(12, seed=5), world=[24, 64, 96], caps_gb=[40, 80, 192],
                       mbs=[1, 2, 4], seq=[4096, 8192], uneven=1, gbs=768),
              mi.Space(models=mi.random_models(8, seed=7), world=[16, 64], caps_gb=[40, 80, 192], mbs=[1, 2, 4],
                       seq=[4096, 8192], uneven=1, stage_max=1)]
    for sp in spaces:
        plan = me.Plan(sp)
        ref = oracle_rows(oracle_mod, sp)
        for mode in (me.ME_OUT_INDEX, me.ME_OUT_FULL, me.ME_OUT_RECORDS):
            res = plan.sweep(mode=mode)
            assert res.status() == 0
            assert_same(me, res, *ref, mode)


@pytest.mark.parametrize("env", [{}, {"ME_K0_BPS": "0"}, {"ME_K0_BPS": "1"}, {"ME_K0_SMEM": "0"},
                                 {"ME_MAX_ROWS": "7"}, {"ME_SERIAL": "1"}, {"ME_K0_FENCE": "0"},
                                 {"ME_K0_FENCE": "0", "ME_K0_SMEM": "0"}],
                         ids=["default", "one-block-per-128-rows", "1bps", "l1", "maxrows7", "serial", "no-fence",
                              "no-fence-l1"])
def test_count_mode_variants(me, oracle_mod, monkeypatch, env):
    """COUNT mode runs K0 alone (grid-stride blocks that stage the sorted u
    lists, totals by atomics): survivor and per-capacity counts equal the
    oracle's for each launch variant, on the whole space and on ragged ranges
    (cut first / last rows go config by config), in paper mode, with a global
    batch, with NEXT-1 and with 8 capacities."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    spaces = [mi.config("C3", uneven=1),
              mi.Space(models=mi.random_models(12, seed=5), world=[24, 64, 96], caps_gb=[40, 80, 192],
                       mbs=[1, 2, 4], seq=[4096, 8192], uneven=1, gbs=768),
              mi.Space(models=mi.random_models(8, seed=7), world=[16, 64], caps_gb=[40, 80, 192], mbs=[1, 2, 4],
                       seq=[4096, 8192], uneven=1, stage_max=1),
              mi.Space(models=mi.random_models(10, seed=11), world=[8, 32, 128], mbs=[1, 2, 3, 5, 8],
                       seq=[2048, 4096, 16384], caps_gb=[16, 24, 40, 48, 80, 94, 141, 192], uneven=1)]
    for sp in spaces:
        plan = me.Plan(sp)
        for b, e in ((0, 0), (13, plan.size - 31), (plan.size // 2, plan.size // 2 + 777)):
            res = plan.sweep(b, e, mode=me.ME_OUT_COUNT)
            assert res.status() == 0
            assert_same(me, res, *oracle_rows(oracle_mod, sp, b, e), me.ME_OUT_COUNT)


@pytest.mark.parametrize("n_mbs,seq", [(1, [4096]), (7, [4096]), (8, [4096]), (9, [4096]), (31, [4096]),
                                       (32, [4096]), (11, [4096, 8192, 16384]), (64, [4096, 8192]),
                                       (43, [4096, 8192, 16384]), (16, [1024, 2048, 4096, 8192, 16384, 32768])],
                         ids=["n1", "n7", "n8", "n9", "n31", "n32", "n33", "n128", "n129", "n96"])
def test_fence_boundaries(me, oracle_mod, n_mbs, seq):
    """K0's search index over each pool's sorted u values (groups of 32,
    blocks of 8; pools over 128 pairs fall back to a plain binary search):
    pools of 1, 7, 8, 9, 31, 32, 33, 96, 128 and 129 pairs, every count and
    every row equal to the oracle's, on the whole space and on a ragged range,
    in COUNT and RECORDS."""
    sp = mi.Space(models=mi.random_models(3, seed=29), world=[8, 16], caps_gb=[24, 40, 80, 192],
                  mbs=list(range(1, n_mbs + 1)), seq=seq, uneven=1)
    plan = me.Plan(sp)
    for b, e in ((0, 0), (5, plan.size - 3)):
        ref = oracle_rows(oracle_mod, sp, b, e)
        for mode in (me.ME_OUT_COUNT, me.ME_OUT_RECORDS):
            res = plan.sweep(b, e, mode=mode)
            assert res.status() == 0
            assert_same(me, res, *ref, mode)


@pytest.mark.parametrize("max_rows", [1, 64, 1000])
def test_subranges_cut_by_rows(me, oracle_mod, monkeypatch, max_rows):
    """Sub-ranges are also cut at max_rows rows (2^21 in production; a small
    cap here, down to one row per sub-range): offsets chain across the cuts
    and the result equals the oracle, for the full range and for ragged
    ranges."""
    monkeypatch.setenv("ME_MAX_ROWS", str(max_rows))
    sp = mi.Space(models=mi.random_models(20, seed=13), world=[16, 48, 64, 128], caps_gb=[40, 80, 192],
                  mbs=[1, 2, 4], seq=[2048, 4096, 8192], uneven=1)
    plan = me.Plan(sp)
    for b, e in ((0, 0), (17, plan.size - 29), (plan.size // 3, plan.size // 3 + 5000)):
        for mode in (me.ME_OUT_INDEX, me.ME_OUT_RECORDS):
            res = plan.sweep(b, e, mode=mode)
            assert res.status() == 0
            assert_same(me, res, *oracle_rows(oracle_mod, sp, b, e or plan.size), mode)


# ---------------------------------------------------------------- NEXT-4: SP off, interleaved 1F1B, byte policies
def test_estimate_variants(me, oracle_mod):
    """me_estimate_batch / me_estimate_stage with the NEXT-4 variants (R28-R30)
    equal the oracle, statuses included"""
    rng = np.random.default_rng(43)
    shapes = mi.random_models(10, seed=47) + [mi.PRESETS["llama3.1-70b"], mi.PRESETS["llama2-13b"]]
    caps = [40 << 30, 80 << 30]
    for shape in shapes:
        cfgs = random_cfgs(rng, shape, 80)
        for cfg in cfgs:
            cfg["sp_off"] = int(rng.integers(0, 2))
            cfg["vpp"] = int(rng.choice([0, 0, 2, 3, 4]))
            cfg["wb"], cfg["gb"], cfg["ob"] = (int(x) for x in rng.choice([(0, 0, 0), (1, 4, 12), (1, 2, 12),
                                                                           (2, 4, 6), (1, 1, 16)]))
            cfg["zero"] = int(rng.integers(0, 4))
            if cfg["vpp"] >= 2 and rng.random() < 0.7:
                cfg.pop("L0", None)
                cfg["uneven"] = 0
                L = shape[2]
                ps = [p for p in range(2, L + 1) if L % (p * cfg["vpp"]) == 0]
                if ps:
                    cfg["p"] = int(rng.choice(ps))
        rows, mask, status = me.me_estimate_batch([shape], None, cfgs, caps_bytes=caps)
        for i, cfg in enumerate(cfgs):
            st = oracle_mod.estimate_status(shape, **cfg)
            assert status[i] == st, (shape, cfg)
            if st == 0:
                e = oracle_mod.estimate(shape, **cfg)
                assert rows[i].tolist() == [e[k] for k in oracle_mod.TERMS], (shape, cfg)
                assert mask[i] == oracle_mod.cap_mask(e["total"], caps)
                if cfg["p"] > 1 and cfg["vpp"] < 2:
                    for stg in (0, cfg["p"] - 1):
                        got, _ = me.me_estimate_stage(shape, stg, **cfg)
                        assert got == oracle_mod.estimate_stage(shape, stg, **cfg), (shape, cfg, stg)


def variant_spaces():
    base = dict(models=mi.random_models(12, seed=53) + [mi.PRESETS["llama3.1-8b"], mi.PRESETS["llama3.1-70b"]],
                world=[16, 24, 64], caps_gb=[24, 40, 80, 192], mbs=[1, 2, 4], seq=[4096, 16384])
    yield "sp_off", mi.Space(**base, sp_off=1, uneven=1)
    yield "sp_off_stage_max", mi.Space(**base, sp_off=1, uneven=1, stage_max=1)
    yield "vpp2", mi.Space(**base, vpp=2)
    yield "vpp3_gbs", mi.Space(**base, vpp=3, gbs=768)
    yield "vpp2_gbs_sp_off", mi.Space(**base, vpp=2, gbs=1536, sp_off=1)
    yield "fp8_weights", mi.Space(**base, wb=1, uneven=1, zero_stage=3)
    yield "bf16_grads_8bit_adam", mi.Space(**base, gb=2, ob=6, gbs=960)


@pytest.mark.parametrize("name,sp", list(variant_spaces()), ids=[n for n, _ in variant_spaces()])
@pytest.mark.parametrize("mode", [0, 1, 3], ids=["count", "index", "records"])
def test_sweep_variants(me, oracle_mod, name, sp, mode):
    plan = me.Plan(sp)
    assert plan.size == oracle_mod.space_size(sp) > 0
    res = plan.sweep(mode=mode)
    assert res.status() == 0
    assert_same(me, res, *oracle_rows(oracle_mod, sp), mode)
    if name in ("vpp2", "vpp3_gbs"):
        # decode agrees on the reduced space
        for i in (0, plan.size // 2, plan.size - 1):
            assert me.me_decode(sp, i)[:2] == oracle_mod.decode(sp, i)[:2]
