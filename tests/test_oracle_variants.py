"""NEXT-4 variants of the oracle (readings R28-R30 in DESIGN.md),
each pinned by a brute-force ledger independent of the oracle's closed forms:

* R28 sequence parallelism off: every saved tensor of P:303-342
  at its per-rank shape under Megatron tensor parallelism without SP -- the
  inputs of the attention and FFN blocks and the RMSNorm inputs whole on
  every TP rank, the rest split by t;
* R29 interleaved 1F1B: a discrete simulation of Megatron's interleaved
  schedule (v model chunks per GPU, warm-up 2(p-1) + (v-1)p forwards on the
  first GPU, chunk of the k-th forward (k mod pv) div p) gives the peak of the
  first GPU's activation bytes over time;
* R30 byte policies: the ledger of P:192-199 with other byte counts per
  parameter (e.g. FP8 weights).
"""
import itertools

import pytest

from test_oracle_ledger import TINY, activation_ledger, numel, one_f_one_b_peak, valid, weight_ledger


def activation_ledger_sp_off(shape, t, c, p, b, s, n_inf, L0, rc=0):
    """Like activation_ledger, with sequence parallelism off: the attention
    input X, the FFN input and the two RMSNorm inputs are whole (not /t); the
    embedding input and the LM head's norm / linear inputs are whole too; the
    FP32 logits stay vocab-parallel (/t)."""
    h, f, L, a, k, v = shape
    hd = h // a
    tok = b * (s // c)
    bf16 = 2
    per_layer = [
        bf16 * tok * h,                                   # X (attention input), whole
        bf16 * tok * h // t, bf16 * tok * hd * k // t, bf16 * tok * hd * k // t,  # Q, K, V
        bf16 * tok * h // t,                              # attention over V output
        bf16 * tok * h,                                   # FFN input, whole
        bf16 * tok * f // t, bf16 * tok * f // t, bf16 * tok * f // t, bf16 * tok * f // t,
        bf16 * tok * h, bf16 * tok * h,                   # RMSNorm inputs, whole
    ]
    if rc:
        layers = n_inf * L0 * bf16 * tok * h + sum(per_layer)
    else:
        layers = n_inf * L0 * sum(per_layer)
    embed = n_inf * 8 * tok * h
    head = 0
    if p == 1:
        head = 4 * tok * v // t + bf16 * tok * h + bf16 * tok * h
    return layers, embed, head


@pytest.mark.parametrize("shape", TINY)
def test_sp_off_matches_ledger(oracle_mod, shape):
    n = 0
    for t, c, p in itertools.product((1, 2, 4), (1, 2), (1, 2, 4)):
        for b, s, rc, dopt in itertools.product((1, 2), (8, 16), (0, 1), (0, 1)):
            if not valid(shape, t, c, p, s):
                continue
            e = oracle_mod.estimate(shape, d=2, t=t, p=p, c=c, b=b, s=s, rc=rc, dopt=dopt, sp_off=1)
            lay, emb, head = activation_ledger_sp_off(shape, t, c, p, b, s, one_f_one_b_peak(p, 4 * p),
                                                      shape[2] // p, rc)
            assert (e["act_layers"], e["act_embed"], e["act_head"]) == (lay, emb, head)
            on = oracle_mod.estimate(shape, d=2, t=t, p=p, c=c, b=b, s=s, rc=rc, dopt=dopt)
            assert (e["params"], e["grads"], e["optim"]) == (on["params"], on["grads"], on["optim"])
            if t == 1:
                assert e == on  # without tensor parallelism SP changes nothing
            else:
                assert e["act_layers"] > on["act_layers"]
            n += 1
    assert n > 20


def interleaved_peak(p, v, m, layer_bytes, embed_bytes, Lc):
    """Megatron's interleaved 1F1B on the first GPU: max over time of the
    bytes of the in-flight chunk-microbatches (Lc layers each) plus the
    embedding inputs of the in-flight microbatches of chunk 0."""
    total = m * v
    W = total if m == p else min(2 * (p - 1) + (v - 1) * p, total)
    live = [0] * v
    best = 0
    f = b = 0

    def fwd():
        nonlocal f
        live[(f % (p * v)) // p] += 1
        f += 1

    def bwd():
        nonlocal b
        live[v - 1 - (b % (p * v)) // p] -= 1
        b += 1

    def mem():
        return sum(live) * Lc * layer_bytes + live[0] * embed_bytes

    for _ in range(W):
        fwd()
        best = max(best, mem())
    for _ in range(total - W):
        fwd()
        best = max(best, mem())
        bwd()
    for _ in range(W):
        bwd()
    assert f == b == total and not any(live)
    return best


@pytest.mark.parametrize("shape", [(16, 24, 8, 4, 2, 32), (32, 48, 12, 8, 4, 64), (24, 40, 16, 4, 4, 48)])
def test_interleaved_matches_schedule_simulation(oracle_mod, shape):
    h, f, L, a, k, v_ = shape
    n = 0
    for p, vpp in itertools.product((2, 3, 4, 6, 8), (2, 3, 4)):
        if L % (p * vpp):
            continue
        Lc = L // (p * vpp)
        for t, c, b, s in itertools.product((1, 2), (1, 2), (1, 2), (8, 16)):
            if not valid(shape, t, c, p, s):
                continue
            # per-microbatch bytes of one layer and of the embedding input (the
            # ledger's, with one layer and one microbatch in flight)
            lay1, emb1, _ = activation_ledger(shape, t, c, p, b, s, 1, 1)
            for gbs in (0, p * 2 * b, p * 4 * b, p * b):
                m = gbs // (2 * b) if gbs else 64 * p
                if gbs and (gbs % (2 * b) or m % p):
                    continue
                e = oracle_mod.estimate(shape, d=2, t=t, p=p, c=c, b=b, s=s, gbs=gbs, vpp=vpp)
                peak = interleaved_peak(p, vpp, m, lay1, emb1, Lc)
                assert e["act_layers"] + e["act_embed"] == peak, (p, vpp, m)
                # both peaks at once (checked by the simulation's joint maximum):
                chunks = p * vpp if m == p else p * vpp + p - 1
                assert e["act_layers"] == chunks * Lc * lay1
                assert e["act_embed"] == min(m, 2 * p) * emb1
                # parameters of the first GPU: v chunks = L/p layers + embedding (Eq.7)
                plain = oracle_mod.estimate(shape, d=2, t=t, p=p, c=c, b=b, s=s, gbs=gbs)
                assert (e["params"], e["grads"], e["optim"]) == (plain["params"], plain["grads"], plain["optim"])
                n += 1
    assert n > 10


def test_interleaved_korthikanti_factor(oracle_mod):
    """paper mode: the first GPU holds L (1 + (p-1)/(p v)) layers' activations
    (Korthikanti et al., cited P:54; non-interleaved: L)"""
    shape = (64, 96, 48, 8, 4, 128)
    for p, vpp in ((2, 2), (4, 2), (4, 3), (6, 4), (8, 3)):
        e = oracle_mod.estimate(shape, d=1, t=1, p=p, c=1, b=1, s=16, vpp=vpp)
        one = oracle_mod.estimate(shape, d=1, t=1, p=p, c=1, b=1, s=16)
        L = shape[2]
        assert e["act_layers"] * p * vpp == one["act_layers"] * (p * vpp + p - 1)
        assert e["act_layers"] * L * p * vpp == one["act_layers"] * (L * p * vpp + L * (p - 1))


def test_interleaved_preconditions(oracle_mod):
    shape = (16, 24, 8, 4, 2, 32)
    assert oracle_mod.estimate_status(shape, d=1, t=1, p=1, c=1, b=1, s=8, vpp=2) == oracle_mod.EDIV
    assert oracle_mod.estimate_status(shape, d=1, t=1, p=2, c=1, b=1, s=8, vpp=3) == oracle_mod.EDIV  # 6 !| 8
    assert oracle_mod.estimate_status(shape, d=2, t=1, p=4, c=1, b=1, s=8, vpp=2, gbs=12) == oracle_mod.EDIV  # m=6
    assert oracle_mod.estimate_status(shape, d=2, t=1, p=4, c=1, b=1, s=8, vpp=2, gbs=16) == 0   # m=8
    assert oracle_mod.estimate_status(shape, d=1, t=1, p=2, c=1, b=1, s=8, vpp=2, uneven=1) == oracle_mod.EINVAL


@pytest.mark.parametrize("shape", TINY[:3])
def test_byte_policies_match_ledger(oracle_mod, shape):
    """R30: weights / gradients / optimizer states at wb / gb / ob bytes per
    parameter (the paper: 2 / 4 / 12); e.g. FP8 weights (wb = 1),
    BF16 gradients (gb = 2), 8-bit Adam moments (ob = 4 + 1 + 1)"""
    h, f, L, a, k, v = shape
    for wb, gb, ob in ((2, 4, 12), (1, 4, 12), (1, 2, 12), (2, 4, 6), (1, 1, 1)):
        for t, c, p, d in itertools.product((1, 2), (1, 2), (1, 2), (1, 3)):
            if not valid(shape, t, c, p, 16):
                continue
            psi = sum(numel(*sh) for _, sh in weight_ledger(shape, t, p, 0))
            chunks = [psi // (d * c) + (1 if r < psi % (d * c) else 0) for r in range(d * c)]
            for dopt, zero in ((0, 0), (1, 0), (1, 2), (1, 3)):
                e = oracle_mod.estimate(shape, d=d, t=t, p=p, c=c, b=1, s=16, dopt=dopt, zero=zero, wb=wb, gb=gb, ob=ob)
                assert e["params"] == wb * (max(chunks) if dopt and zero >= 3 else psi)
                assert e["grads"] == gb * (max(chunks) if dopt and zero >= 2 else psi)
                assert e["optim"] == ob * (max(chunks) if dopt else psi)
                if (wb, gb, ob) == (2, 4, 12):
                    assert e == oracle_mod.estimate(shape, d=d, t=t, p=p, c=c, b=1, s=16, dopt=dopt, zero=zero)
