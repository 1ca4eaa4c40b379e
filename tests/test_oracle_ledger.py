"""Brute-force pins for each oracle term separately (CPU only).

The paper's tables only print totals.  Here each term is rebuilt from first
principles on tiny models, independently of the oracle's closed forms:

* parameters: every weight tensor of a Llama decoder with Megatron's split rule
  (column-parallel Q/K/V/up/gate, row-parallel O/down, vocab-parallel embedding
  and LM head, replicated RMSNorms; Fig.1-3 text P:145-183) placed on
  pipeline stage 0, counted element by element for TP rank 0;
* optimizer shard: Psi_s parameters dealt to d*c ranks in contiguous chunks and
  the largest chunk taken (reading R8);
* activations: every tensor the paper lists as saved with its
  per-rank shape under SP/TP/CP, summed over the microbatches a discrete
  1F1B schedule (PipeDream / Megatron non-interleaved) keeps
  in flight on stage 0.
"""
import itertools

import pytest

import me_inputs as mi

TINY = [(16, 24, 4, 4, 2, 32), (32, 48, 8, 8, 4, 64), (24, 40, 6, 4, 4, 48),
        (64, 96, 8, 8, 1, 128), (16, 16, 3, 2, 2, 16)]


def numel(*shape):
    n = 1
    for x in shape:
        n *= x
    return n


def stage_layers(L, p, L0=None):
    """Layer ids held by each pipeline stage: L/p each; uneven splits give
    stage 0 ceil(L/p) (R19) and the rest as evenly as possible."""
    if L0 is None:
        L0 = -(-L // p)
    rest = L - L0
    out = [list(range(L0))]
    nxt = L0
    for i in range(1, p):
        k = rest // (p - 1) + (1 if (i - 1) < rest % (p - 1) else 0)
        out.append(list(range(nxt, nxt + k)))
        nxt += k
    assert nxt == L
    return out


def weight_ledger(shape, t, p, stage, L0=None):
    """All weight tensors on (tp rank 0, pipeline stage `stage`), as shapes."""
    h, f, L, a, k, v = shape
    hd = h // a
    tensors = []
    layers = stage_layers(L, p, L0)[stage]
    for _ in layers:
        tensors += [
            ("W_Q", (h, h // t)),              # column-parallel
            ("W_K", (h, hd * k // t)),          # column-parallel, GQA (h, h/g)
            ("W_V", (h, hd * k // t)),
            ("W_O", (h // t, h)),               # row-parallel
            ("W_up", (h, f // t)), ("W_gate", (h, f // t)),  # column-parallel
            ("W_down", (f // t, h)),            # row-parallel
            ("input_norm", (h,)), ("post_attn_norm", (h,)),  # replicated (R6)
        ]
    if stage == 0:
        tensors.append(("embedding", (v // t, h)))       # vocab-parallel
    if stage == p - 1:
        tensors.append(("final_norm", (h,)))
        tensors.append(("lm_head", (h, v // t)))         # untied
    return tensors


def one_f_one_b_peak(p, m, stage=0):
    """Discrete non-interleaved 1F1B: warm-up forwards, steady 1F1B, cool-down
    backwards; returns the max number of microbatches whose activations the
    stage holds at once."""
    warm = min(p - stage - 1, m)
    ops = ["F"] * warm
    for _ in range(m - warm):
        ops += ["F", "B"]
    ops += ["B"] * warm
    live = peak = 0
    for op in ops:
        live += 1 if op == "F" else -1
        peak = max(peak, live)
    assert live == 0 and ops.count("F") == m
    return peak


def activation_ledger(shape, t, c, p, b, s, n_inf, L0, rc=0):
    """Bytes of every saved activation on stage 0, TP rank 0 (SP on, CP on)."""
    h, f, L, a, k, v = shape
    hd = h // a
    tok = b * (s // c)               # tokens of one microbatch on this CP rank
    bf16 = 2
    per_layer = [
        # attention block: X, Q, K, V, attention output; QK^T and
        # softmax store nothing under FlashAttention-2
        bf16 * tok * h // t, bf16 * tok * h // t, bf16 * tok * hd * k // t,
        bf16 * tok * hd * k // t, bf16 * tok * h // t,
        # FFN: input, up out, gate out, activation out, down input
        bf16 * tok * h // t, bf16 * tok * f // t, bf16 * tok * f // t, bf16 * tok * f // t,
        bf16 * tok * f // t,
        # two RMSNorm inputs
        bf16 * tok * h // t, bf16 * tok * h // t,
    ]
    if rc:
        # R20: only each layer's input is kept, plus one layer's full set while
        # it is recomputed in the backward pass
        layers = n_inf * L0 * bf16 * tok * h // t + sum(per_layer)
    else:
        layers = n_inf * L0 * sum(per_layer)
    # embedding input, literal Eq.13 (R13 keeps the printed h)
    embed = n_inf * 8 * tok * h // t
    head = 0
    if p == 1:
        # Eq.14: FP32 logits, output-norm input, LM-head input
        head = 4 * tok * v // t + bf16 * tok * h // t + bf16 * tok * h // t
    return layers, embed, head


def valid(shape, t, c, p, s, uneven=False):
    h, f, L, a, k, v = shape
    return (k % t == 0 and v % t == 0 and f % t == 0 and s % c == 0 and p <= L
            and (uneven or L % p == 0))


@pytest.mark.parametrize("shape", TINY)
def test_ledger_matches_oracle_terms(oracle_mod, shape):
    n = 0
    for N in (1, 2, 4, 6, 8, 12, 16):
        for t, c, p in itertools.product(range(1, 17), repeat=3):
            if N % (t * c * p):
                continue
            d = N // (t * c * p)
            for b, s, rc, dopt in itertools.product((1, 2), (8, 16, 24), (0, 1), (0, 1)):
                if not valid(shape, t, c, p, s):
                    continue
                e = oracle_mod.estimate(shape, d=d, t=t, p=p, c=c, b=b, s=s, rc=rc, dopt=dopt)
                psi = sum(numel(*sh) for _, sh in weight_ledger(shape, t, p, 0))
                assert e["params"] == 2 * psi and e["grads"] == 4 * psi
                chunks = [psi // (d * c) + (1 if r < psi % (d * c) else 0) for r in range(d * c)]
                assert sum(chunks) == psi
                assert e["optim"] == (12 * max(chunks) if dopt else 12 * psi)
                n_inf = one_f_one_b_peak(p, m=4 * p)  # paper mode: m >= p (R17)
                L0 = shape[2] // p
                lay, emb, head = activation_ledger(shape, t, c, p, b, s, n_inf, L0, rc)
                assert (e["act_layers"], e["act_embed"], e["act_head"]) == (lay, emb, head)
                assert e["total"] == 6 * psi + e["optim"] + lay + emb + head
                n += 1
    assert n > 100


@pytest.mark.parametrize("shape", TINY[:3])
def test_ledger_gbs_and_uneven(oracle_mod, shape):
    """R17 (in-flight microbatches from a global batch) and R19 (uneven PP)."""
    h, f, L, a, k, v = shape
    n = 0
    for t, c, p, d in itertools.product((1, 2), (1, 2), range(1, L + 1), (1, 2, 3)):
        for b, s, gbs in itertools.product((1, 2), (8, 16), (0, 6, 12, 24, 48)):
            if not valid(shape, t, c, p, s, uneven=True):
                continue
            if gbs and gbs % (d * b):
                continue
            e = oracle_mod.estimate(shape, d=d, t=t, p=p, c=c, b=b, s=s, gbs=gbs, uneven=1)
            m = gbs // (d * b) if gbs else 4 * p
            n_inf = one_f_one_b_peak(p, m)
            L0 = L if p == 1 else -(-L // p)
            psi = sum(numel(*sh) for _, sh in weight_ledger(shape, t, p, 0, L0))
            assert e["params"] == 2 * psi
            lay, emb, head = activation_ledger(shape, t, c, p, b, s, n_inf, L0)
            assert (e["act_layers"], e["act_embed"], e["act_head"]) == (lay, emb, head)
            n += 1
    assert n > 50


def test_one_f_one_b_closed_form():
    """Stage i of 1F1B holds min(m, p - i) microbatches."""
    for p in range(1, 17):
        for m in range(1, 65):
            for i in range(p):
                assert one_f_one_b_peak(p, m, i) == min(m, p - i)


@pytest.mark.parametrize("shape", TINY)
def test_partition_identity(shape):
    """Corrected SPEC S:92 (reading R25): summing every stage's TP-rank-0 shard
    times t over-counts exactly the replicated norms, (t-1)(2hL + h)."""
    h, f, L, a, k, v = shape
    psi_total = sum(numel(*sh) for _, sh in weight_ledger(shape, 1, 1, 0))
    for t in (1, 2):
        for p in range(1, L + 1):
            if L % p or k % t or f % t or v % t:
                continue
            s = sum(numel(*sh) for st in range(p) for _, sh in weight_ledger(shape, t, p, st))
            assert t * s - (t - 1) * (2 * h * L + h) == psi_total


def test_total_params_from_ledger(oracle_mod):
    for shape in TINY + [mi.PRESETS["llama3.1-8b"], mi.PRESETS["llama2-7b"]]:
        psi = sum(numel(*sh) for _, sh in weight_ledger(shape, 1, 1, 0))
        assert oracle_mod.total_params(shape) == psi
        assert oracle_mod.stage0_params(shape, 1, 1, shape[2]) == psi


def compositions(L, p):
    """every split of L layers into p stages of >= 1 layer (brute force)"""
    if p == 1:
        yield (L,)
        return
    for first in range(1, L - p + 2):
        for rest in compositions(L - first, p - 1):
            yield (first,) + rest


def test_uneven_first_stage_is_the_worst_case(oracle_mod):
    """R19 (uneven PP, not in the paper): over every split of L layers into p
    stages, ceil(L/p) is the smallest possible largest stage, so a balanced
    split has a stage of ceil(L/p) layers; the oracle puts it first, where the
    1F1B schedule keeps the most microbatches (p - i on stage i), so its
    stage-0 layer activations bound every stage of every balanced split.  The
    oracle's own split of the remaining layers is balanced (its largest stage
    is stage 0)."""
    shape = (16, 24, 14, 4, 2, 32)
    for L in range(1, 15):
        for p in range(1, L + 1):
            splits = list(compositions(L, p))
            best = min(max(s) for s in splits)
            assert best == -(-L // p)
            L0 = oracle_mod.first_stage_layers(shape[:2] + (L,) + shape[3:], d=1, t=1, p=p, c=1, b=1, s=8, uneven=1)
            assert L0 == best
            balanced = [s for s in splits if max(s) == best]
            worst = max(max((p - i) * s[i] for i in range(p)) for s in balanced)
            assert worst == p * L0  # stage 0 holding ceil(L/p) layers with p microbatches in flight
            mine = tuple(len(x) for x in stage_layers(L, p))
            assert mine in balanced and mine[0] == L0
            if p > 1:
                cfg = dict(d=1, t=1, p=p, c=1, b=1, s=8, uneven=1)
                m = shape[:2] + (L,) + shape[3:]
                for i in range(p):
                    assert oracle_mod.stage_layers(m, i, **cfg) == mine[i]
