"""NEXT-1 (per-stage estimator, max over stages): oracle pins (CPU only).

Stage i holds Eq.7 / Eq.8 / Eq.9 parameters for its layers and the
activations of min(m, p - i) in-flight microbatches (1F1B);
the embedding input lives on stage 0, the LM head on the last stage.  Pinned by
the brute-force tensor ledger of tests/test_oracle_ledger.py run per stage, the
identity with the stage-0 estimator, the corrected partition identity and the
example of SURVEY §0 finding 8."""
import itertools

import numpy as np
import pytest

import me_inputs as mi
from test_oracle_ledger import TINY, activation_ledger, numel, one_f_one_b_peak, stage_layers, weight_ledger


def stage_ledger(shape, t, c, p, b, s, stage, m, rc=0, L0=None):
    """Bytes on (tp rank 0, stage) from the tensor ledgers."""
    h, f, L, a, k, v = shape
    layers = stage_layers(L, p, L0)[stage]
    psi = sum(numel(*sh) for _, sh in weight_ledger(shape, t, p, stage, L0))
    n = one_f_one_b_peak(p, m, stage)
    lay, emb, _ = activation_ledger(shape, t, c, p, b, s, n, len(layers), rc)
    tok = b * (s // c)
    head = (4 * tok * v // t + 4 * tok * h // t) * n if stage == p - 1 else 0
    return psi, lay, emb if stage == 0 else 0, head


@pytest.mark.parametrize("shape", TINY)
def test_stage_terms_match_ledger(oracle_mod, shape):
    h, f, L, a, k, v = shape
    n = 0
    for t, c, p, d in itertools.product((1, 2), (1, 2), range(1, L + 1), (1, 3)):
        for b, s, gbs, rc, dopt in itertools.product((1, 2), (8, 16), (0, 12, 48), (0, 1), (0, 1)):
            if k % t or v % t or f % t or s % c or (gbs and gbs % (d * b)):
                continue
            cfg = dict(d=d, t=t, p=p, c=c, b=b, s=s, gbs=gbs, rc=rc, dopt=dopt, uneven=1)
            m = gbs // (d * b) if gbs else 4 * p
            L0 = L if p == 1 else -(-L // p)
            for i in range(p):
                e = oracle_mod.estimate_stage(shape, i, **cfg)
                psi, lay, emb, head = stage_ledger(shape, t, c, p, b, s, i, m, rc, L0)
                assert e["params"] == 2 * psi and e["grads"] == 4 * psi
                assert e["optim"] == (12 * -(-psi // (d * c)) if dopt else 12 * psi)
                assert (e["act_layers"], e["act_embed"], e["act_head"]) == (lay, emb, head), (cfg, i)
                n += 1
    assert n > 200


def test_stage0_is_the_paper_estimate(oracle_mod):
    rng = np.random.default_rng(5)
    for shape in mi.random_models(20, seed=3):
        h, f, L, a, k, v = shape
        for _ in range(20):
            p = int(rng.integers(1, L + 1))
            cfg = dict(d=int(rng.integers(1, 9)), t=1, p=p, c=1, b=int(rng.integers(1, 5)), s=4096,
                       rc=int(rng.integers(0, 2)), dopt=int(rng.integers(0, 2)), uneven=1)
            assert oracle_mod.estimate_stage(shape, 0, **cfg) == oracle_mod.estimate(shape, **cfg)


def test_stage_partition_identity(oracle_mod):
    """Corrected SPEC S:92 (R25) on the per-stage parameter counts."""
    for shape in TINY + [mi.PRESETS["llama3.1-8b"]]:
        h, f, L, a, k, v = shape
        psi = oracle_mod.total_params(shape)
        for t in (1, 2, 4):
            if k % t or v % t or f % t:
                continue
            for p in range(1, L + 1):
                cfg = dict(d=1, t=t, p=p, c=1, b=1, s=8, uneven=1)
                tot = sum(oracle_mod.estimate_stage(shape, i, **cfg)["params"] // 2 for i in range(p))
                assert t * tot - (t - 1) * (2 * h * L + h) == psi


def test_middle_stages_never_exceed_stage0(oracle_mod):
    """The property the GPU path relies on: max over stages = max(stage 0, last)."""
    rng = np.random.default_rng(9)
    for shape in mi.random_models(30, seed=4):
        h, f, L, a, k, v = shape
        for _ in range(10):
            p = int(rng.integers(2, L + 1)) if L > 1 else 1
            gbs = int(rng.choice([0, 64, 1024]))
            d, b = int(rng.choice([1, 2, 4])), int(rng.choice([1, 2]))
            if gbs and gbs % (d * b):
                gbs = 0
            cfg = dict(d=d, t=1, p=p, c=1, b=b, s=4096, gbs=gbs, rc=int(rng.integers(0, 2)),
                       dopt=int(rng.integers(0, 2)), uneven=1)
            tot = [oracle_mod.estimate_stage(shape, i, **cfg)["total"] for i in range(p)]
            assert max(tot[1:-1] or [0]) <= tot[0]
            e, arg = oracle_mod.estimate_max(shape, **cfg)
            assert e["total"] == max(tot) and arg == tot.index(max(tot))


def test_last_stage_can_dominate(oracle_mod):
    """SURVEY §0 finding 8: h=1024, L=16, GQA 8/8, h_ffn=2816, v=256000, p=2,
    s=4096, b=1 -- the last stage holds 2.10x the stage-0 activation bytes."""
    shape = (1024, 2816, 16, 8, 8, 256000)
    cfg = dict(d=1, t=1, p=2, c=1, b=1, s=4096)
    s0 = oracle_mod.estimate_stage(shape, 0, **cfg)
    s1 = oracle_mod.estimate_stage(shape, 1, **cfg)
    act = lambda e: e["act_layers"] + e["act_embed"] + e["act_head"]  # noqa: E731
    assert round(act(s1) / act(s0), 2) == 2.10
    e, arg = oracle_mod.estimate_max(shape, **cfg)
    assert arg == 1 and e == s1
