"""Oracle invariants and the canonical enumeration order (CPU only).

Properties are the ones SPEC states for the method plus the
identities of DESIGN.md §3 readings R8/R17/R20/R21; the enumeration is checked
against an itertools re-statement of the canonical order and
the closed-form tuple counts of the configs."""
import itertools

import numpy as np

import pytest

import me_inputs as mi

M8 = mi.PRESETS["llama3.1-8b"]
M70 = mi.PRESETS["llama3.1-70b"]


def est(o, shape, **kw):
    base = dict(d=1, t=1, p=1, c=1, b=1, s=8192)
    base.update(kw)
    return o.estimate(shape, **base)


def test_spec_worked_examples(oracle_mod):
    o = oracle_mod
    # SPEC S:57
    assert o.attention_params(M8) == 41_943_040
    assert o.ffn_params(M8) == 176_160_768
    assert o.total_params(M8) == 8_030_261_248
    assert o.total_params(M70) == 70_553_706_496
    assert o.stage0_params(M8, 4, 2, 16) == 1_003_880_448
    e = est(o, M8, t=4, p=2)
    assert e["params"] + e["grads"] + e["optim"] == 18_069_848_064
    assert o.activation_per_layer(M8, 8192, 1) == 1_375_731_712
    e = est(o, M8, d=2, t=2)
    assert e["act_layers"] + e["act_embed"] + e["act_head"] == 24_314_380_288
    e = est(o, M8, t=4, p=2)
    assert e["act_layers"] + e["act_embed"] + e["act_head"] == 11_140_071_424
    # trivial cases of Eq.1/2
    assert o.attention_params((4, 4, 1, 2, 2, 4)) == 4 * 16          # k = a -> 4h^2
    assert o.ffn_params((2, 3, 1, 1, 1, 1)) == 18


def test_public_parameter_counts(oracle_mod):
    """Eq.3 reproduces the widely published parameter counts (external pin, R26)."""
    pub = {"llama2-7b": 6_738_415_616, "llama2-13b": 13_015_864_320,
           "llama2-70b": 68_976_648_192, "llama3.1-8b": 8_030_261_248,
           "llama3.1-70b": 70_553_706_496}
    for name, n in pub.items():
        assert oracle_mod.total_params(mi.PRESETS[name]) == n


def test_degenerate_single_gpu(oracle_mod):
    """t=c=p=d=1: 18 Psi (Eq.4 ledger) + activations of the single stage."""
    o = oracle_mod
    for shape in (M8, M70, mi.PRESETS["llama2-7b"]):
        e = est(o, shape, s=4096)
        assert e["params"] + e["grads"] + e["optim"] == 18 * o.total_params(shape)
        h, f, L, a, k, v = shape
        assert e["act_layers"] == L * o.activation_per_layer(shape, 4096, 1)


def test_monotonic_and_linear(oracle_mod):
    o = oracle_mod
    for b, s in ((1, 4096), (2, 8192)):
        base = est(o, M8, d=2, t=2, p=2, c=2, b=b, s=s)
        # doubling c strictly decreases the total
        assert est(o, M8, d=2, t=2, p=2, c=4, b=b, s=s)["total"] < base["total"]
        # doubling d shrinks model states only
        e = est(o, M8, d=4, t=2, p=2, c=2, b=b, s=s)
        assert e["optim"] < base["optim"] and e["params"] == base["params"]
        assert (e["act_layers"], e["act_embed"]) == (base["act_layers"], base["act_embed"])
        # larger t never increases any term
        e = est(o, M8, d=2, t=4, p=2, c=2, b=b, s=s)
        for k in ("params", "optim", "act_layers", "act_embed", "total"):
            assert e[k] <= base[k]
    # activations are linear in s and b
    e1, e2 = est(o, M8, t=2, p=2, b=1, s=4096), est(o, M8, t=2, p=2, b=3, s=8192)
    for k in ("act_layers", "act_embed", "act_head"):
        assert e2[k] == 6 * e1[k]


def test_first_stage_independent_of_p(oracle_mod):
    """Layer activations on stage 0 do not depend on p; the embedding term grows
    as 8 sbh p / (tc)."""
    o = oracle_mod
    ref = est(o, M8, t=2, p=2, c=1)
    for p in (2, 4, 8, 16, 32):
        e = est(o, M8, t=2, p=p, c=1)
        assert e["act_layers"] == ref["act_layers"]
        assert e["act_embed"] - ref["act_embed"] == 8192 * 4096 // 2 * 8 * (p - 2)


def test_extension_identities(oracle_mod):
    o = oracle_mod
    for shape in (M8, M70):
        for d, t, p, c in ((1, 2, 2, 1), (4, 2, 4, 2), (3, 1, 2, 1)):
            kw = dict(d=d, t=t, p=p, c=c, b=2, s=8192)
            on, off = est(o, shape, **kw), est(o, shape, dopt=0, **kw)
            # R21: distributed optimizer off = Eq.4 (12 Psi_s unsharded)
            assert off["optim"] == 12 * on["params"] // 2
            if d * c == 1:
                assert off == on
            # R20: recompute keeps layer inputs for n_inf L0 (layer, mb) pairs
            # plus one full layer
            rc = est(o, shape, rc=1, **kw)
            h, f, L, a, k, v = shape
            n_inf_L0 = p * (L // p)
            u = 8192 // c * 2
            assert rc["act_layers"] == 2 * u * (h // t) * n_inf_L0 + on["act_layers"] // n_inf_L0
            # R8 ceil: exact when (d c) | Psi_s, otherwise within 12 * 1 parameter
            psi = on["params"] // 2
            assert on["optim"] == 12 * (-(-psi // (d * c)))
    # the R8 example of DESIGN.md: 8B, N = 24, t = c = p = 1
    assert est(o, M8, d=24)["optim"] == 4_015_130_628


def test_gbs_in_flight(oracle_mod):
    """R17: with m = gbs/(d b) < p only m microbatches are in flight; gbs = 1024
    reproduces paper mode in every paper cell (m >= p there)."""
    o = oracle_mod
    paper = est(o, M8, d=8, t=1, p=4, b=1)
    assert est(o, M8, d=8, t=1, p=4, b=1, gbs=1024) == paper
    small = est(o, M8, d=8, t=1, p=4, b=1, gbs=16)  # m = 2
    assert small["act_embed"] * 2 == paper["act_embed"]
    assert small["act_layers"] * 2 == paper["act_layers"]


def test_preconditions(oracle_mod):
    o = oracle_mod
    EINVAL, EDIV = o.EINVAL, o.EDIV
    st = o.estimate_status
    assert st((4096, 14336, 32, 32, 7, 128256), d=1, t=1, p=1, c=1, b=1, s=8) == EINVAL  # k∤a
    assert st((4000, 14336, 32, 64, 8, 128256), d=1, t=1, p=1, c=1, b=1, s=8) == EINVAL  # a∤h
    assert st(M8, d=0, t=1, p=1, c=1, b=1, s=8) == EINVAL
    assert st(M8, d=1, t=16, p=1, c=1, b=1, s=8192) == EDIV    # t ∤ k
    assert st(M8, d=1, t=3, p=1, c=1, b=1, s=8192) == EDIV
    assert st(M8, d=1, t=1, p=1, c=3, b=1, s=8192) == EDIV     # c ∤ s
    assert st(M8, d=1, t=1, p=33, c=1, b=1, s=8192) == EDIV    # p > L
    assert st(M8, d=1, t=1, p=3, c=1, b=1, s=8192) == EDIV     # p ∤ L, even split
    assert st(M8, d=1, t=1, p=3, c=1, b=1, s=8192, uneven=1) == 0
    assert o.first_stage_layers(M8, d=1, t=1, p=3, c=1, b=1, s=8192, uneven=1) == 11
    assert st(M8, d=3, t=1, p=1, c=1, b=1, s=8192, gbs=1024) == EDIV  # (d b) ∤ gbs
    assert st(M8, d=1, t=1, p=2, c=1, b=1, s=8192, L0=32) == EDIV     # no layer left for stage 1
    assert st(M8, d=1, t=1, p=2, c=1, b=1, s=8192, L0=31) == 0
    assert st(M8, d=1, t=1, p=2, c=1, b=1, s=8192, L0=30) == 0


def canonical(sp):
    """The canonical order of DESIGN.md §4, restated with itertools."""
    for mi_, m in enumerate(sp.models):
        h, f, L, a, k, v = m
        for N in sp.world:
            for t, c, p in itertools.product(range(1, N + 1), repeat=3):
                if N % (t * c * p):
                    continue
                d = N // (t * c * p)
                if k % t or v % t or f % t or p > L or (not sp.uneven and L % p):
                    continue
                if (sp.max_t and t > sp.max_t) or (sp.max_c and c > sp.max_c) or \
                        (sp.max_p and p > sp.max_p) or (sp.gpus_per_node and t > sp.gpus_per_node):
                    continue
                for b, s in itertools.product(sp.mbs, sp.seq):
                    if s % c or (sp.gbs and sp.gbs % (d * b)):
                        continue
                    for rc in (0, 1):
                        if not (sp.rc_mask >> rc) & 1:
                            continue
                        for dopt in (0, 1):
                            if (sp.do_mask >> dopt) & 1:
                                yield mi_, N, dict(d=d, t=t, p=p, c=c, b=b, s=s, gbs=sp.gbs,
                                                   rc=rc, dopt=dopt)


def small_spaces():
    yield mi.config("C1")
    yield mi.Space(models=mi.random_models(3, seed=7, small=True), world=[6, 8, 12],
                   caps_gb=[1], mbs=[1, 3], seq=[8, 12], gbs=24, uneven=1, rc_mask=2, do_mask=3)
    yield mi.Space(models=[(16, 24, 4, 4, 2, 32), (32, 48, 8, 8, 4, 64)], world=[16, 4],
                   caps_gb=[1, 2], mbs=[2, 1], seq=[16, 8], max_t=4, max_p=2, gpus_per_node=2,
                   rc_mask=1, do_mask=2)


@pytest.mark.parametrize("sp", list(small_spaces()), ids=lambda s: s.name or "rand")
def test_enumeration_order(oracle_mod, sp):
    ref = list(canonical(sp))
    assert oracle_mod.space_size(sp) == len(ref)
    for i in list(range(0, len(ref), max(1, len(ref) // 97))) + [len(ref) - 1]:
        mid, N, cfg = oracle_mod.decode(sp, i)
        rm, rN, rc = ref[i]
        assert (mid, N) == (rm, rN) and {k: cfg[k] for k in rc} == rc, i
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.decode(sp, len(ref))


def test_space_sizes_closed_form(oracle_mod):
    # C1: the 20 ordered factorisations of 8 into (d, t, p, c) x 3 mbs x 4 (rc, do)
    assert oracle_mod.space_size(mi.config("C1")) == 20 * 3 * 4
    # C3: t = 2^i (i<4), p = 2^j (p | 80, j<5), c | 1024/(t p): 11 - i - j choices;
    # uneven PP adds p = 32, 64
    n = sum(11 - i - j for i in range(4) for j in range(5))
    assert n == 150
    assert oracle_mod.space_size(mi.config("C3")) == n * 16 * 6 * 4
    n_u = n + sum(11 - i - j for i in range(4) for j in (5, 6))
    assert oracle_mod.space_size(mi.config("C3", uneven=1)) == n_u * 16 * 6 * 4


def test_sweep_matches_pointwise(oracle_mod):
    sp = mi.config("C1")
    idx, rows, n, caps = oracle_mod.sweep(sp)
    ref = []
    for i, (mid, N, cfg) in enumerate(canonical(sp)):
        e = oracle_mod.estimate(sp.models[mid], **cfg)
        mask = oracle_mod.cap_mask(e["total"], sp.cap_bytes)
        if mask:
            ref.append((i | (mask << 56), [e[k] for k in oracle_mod.TERMS]))
    assert n == len(ref) and list(idx) == [r[0] for r in ref]
    assert rows.tolist() == [r[1] for r in ref]
    # threads do not change the result
    idx2, rows2, n2, caps2 = oracle_mod.sweep(sp, threads=5)
    assert (idx2 == idx).all() and (rows2 == rows).all() and caps2 == caps
    # sub-ranges concatenate
    a = oracle_mod.sweep(sp, 0, 77)[0]
    b = oracle_mod.sweep(sp, 77, 240)[0]
    assert list(a) + list(b) == list(idx)


def test_points_match_sweep(oracle_mod):
    sp = mi.config("C3")
    idx, rows, n, caps = oracle_mod.sweep(sp)
    index = (idx & np.uint64((1 << 56) - 1))
    pick = index[::97]
    r2, m2 = oracle_mod.points(sp, pick[::-1])
    assert (r2[::-1] == rows[::97]).all()
    assert (m2[::-1] == (idx[::97] >> np.uint64(56))).all()


def test_zero_stages(oracle_mod):
    """NEXT-4 byte policies: ZeRO stage 1 (the paper's distributed optimizer),
    2 (+ FP32 gradients) and 3 (+ BF16 weights) sharded over d*c.  Pins: the
    ZeRO per-device model-state formulas (P:53, P:188 cite ZeRO) with this
    ledger's FP32 gradients -- stage 1: (2 + 4) Psi + 12 Psi / N_d, stage 2:
    2 Psi + (4 + 12) Psi / N_d, stage 3: (2 + 4 + 12) Psi / N_d -- exact when
    N_d = d c divides Psi, the largest contiguous shard otherwise; stage 1 is
    the paper's estimate; N_d = 1 reduces every stage to Eq.4."""
    o = oracle_mod
    for shape in (M8, M70, (16, 24, 4, 4, 2, 32)):
        for d, t, p, c in ((1, 1, 1, 1), (8, 1, 1, 1), (4, 2, 2, 2), (3, 1, 2, 1), (5, 2, 1, 1)):
            kw = dict(d=d, t=t, p=p, c=c, b=1, s=16)
            base = o.estimate(shape, **kw)
            psi = base["params"] // 2
            nd = d * c
            share = -(-psi // nd)
            assert o.estimate(shape, zero=1, **kw) == base
            z2 = o.estimate(shape, zero=2, **kw)
            z3 = o.estimate(shape, zero=3, **kw)
            assert (z2["params"], z2["grads"], z2["optim"]) == (2 * psi, 4 * share, 12 * share)
            assert (z3["params"], z3["grads"], z3["optim"]) == (2 * share, 4 * share, 12 * share)
            if psi % nd == 0:
                assert 18 * psi == (z3["params"] + z3["grads"] + z3["optim"]) * nd
                assert z2["params"] + z2["grads"] + z2["optim"] == 2 * psi + 16 * psi // nd
            for z in (z2, z3):  # activations untouched
                assert (z["act_layers"], z["act_embed"], z["act_head"]) == \
                    (base["act_layers"], base["act_embed"], base["act_head"])
            if nd == 1:
                assert z2 == base and z3 == base
            # without the distributed optimizer the stage is irrelevant (Eq.4)
            off = o.estimate(shape, dopt=0, **kw)
            assert o.estimate(shape, dopt=0, zero=3, **kw) == off
