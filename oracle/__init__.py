"""CPU oracle for the arXiv 2411.06465 memory estimator (ctypes over
oracle/me_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product
package paper_2411_06465_b200 never imports it, and it never imports the
product.  Parity status per function is listed in DESIGN.md §3 ("parity
unpinned" for readings R8, R19, R20 beyond their reductions to the paper).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "me_oracle.c"
LIB = HERE / "libme_oracle.so"

OK, EINVAL, EDIV, EOVERFLOW, ENOMEM, ERANGE = 0, 1, 2, 3, 4, 7


class OracleError(RuntimeError):
    def __init__(self, status, what=""):
        super().__init__(f"oracle status {status} {what}")
        self.status = status


def build(force: bool = False) -> Path:
    if force or not LIB.exists() or LIB.stat().st_mtime < max(SRC.stat().st_mtime,
                                                               (HERE / "me_oracle.h").stat().st_mtime):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-Wall", "-shared", "-fPIC", "-pthread",
                               str(SRC), "-o", str(LIB)])
    return LIB


class Model(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in ("h", "f", "L", "a", "k", "v")]


class Cfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in ("d", "t", "p", "c", "b", "s", "gbs", "L0")] + [
        ("rc", ctypes.c_uint8), ("dopt", ctypes.c_uint8), ("uneven", ctypes.c_uint8),
        ("zero", ctypes.c_uint8), ("sp_off", ctypes.c_uint8), ("vpp", ctypes.c_uint8), ("wb", ctypes.c_uint8),
        ("gb", ctypes.c_uint8), ("ob", ctypes.c_uint8)]


class Breakdown(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in
                ("params", "grads", "optim", "act_layers", "act_embed", "act_head", "total")]


TERMS = ("params", "grads", "optim", "act_layers", "act_embed", "act_head", "total")

_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)


class SpaceC(ctypes.Structure):
    _fields_ = [("models", ctypes.POINTER(Model)), ("n_models", ctypes.c_uint32),
                ("world", _u32p), ("n_world", ctypes.c_uint32),
                ("cap_bytes", _u64p), ("n_caps", ctypes.c_uint32),
                ("gpus_per_node", ctypes.c_uint32),
                ("mbs", _u32p), ("n_mbs", ctypes.c_uint32),
                ("seq", _u32p), ("n_seq", ctypes.c_uint32),
                ("rc_mask", ctypes.c_uint8), ("do_mask", ctypes.c_uint8),
                ("uneven", ctypes.c_uint8), ("stage_max", ctypes.c_uint8),
                ("gbs", ctypes.c_uint32), ("max_t", ctypes.c_uint32), ("max_c", ctypes.c_uint32),
                ("max_p", ctypes.c_uint32), ("thr_num", ctypes.c_uint32),
                ("thr_den", ctypes.c_uint32), ("zero_stage", ctypes.c_uint32),
                ("sp_off", ctypes.c_uint8), ("vpp", ctypes.c_uint8), ("wb", ctypes.c_uint8), ("gb", ctypes.c_uint8),
                ("ob", ctypes.c_uint8), ("_pad", ctypes.c_uint8 * 3)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(str(build()))
        P = ctypes.POINTER
        for name in ("or_attention_params", "or_ffn_params", "or_total_params"):
            getattr(_lib, name).argtypes = [P(Model), _u64p]
        _lib.or_stage0_params.argtypes = [P(Model), ctypes.c_uint32, ctypes.c_uint32,
                                          ctypes.c_uint32, _u64p]
        _lib.or_activation_per_layer.argtypes = [P(Model), ctypes.c_uint32, ctypes.c_uint32, _u64p]
        _lib.or_first_stage_layers.argtypes = [P(Model), P(Cfg)]
        _lib.or_first_stage_layers.restype = ctypes.c_uint32
        _lib.or_estimate.argtypes = [P(Model), P(Cfg), P(Breakdown)]
        _lib.or_cap_mask.argtypes = [ctypes.c_uint64, _u64p, ctypes.c_uint32, ctypes.c_uint32,
                                     ctypes.c_uint32]
        _lib.or_cap_mask.restype = ctypes.c_uint32
        _lib.or_space_size.argtypes = [P(SpaceC), _u64p]
        _lib.or_decode.argtypes = [P(SpaceC), ctypes.c_uint64, _u32p, _u32p, P(Cfg)]
        _lib.or_sweep.argtypes = [P(SpaceC), ctypes.c_uint64, ctypes.c_uint64, _u64p,
                                  P(Breakdown), ctypes.c_uint64, _u64p, _u64p, ctypes.c_int]
        _lib.or_points.argtypes = [P(SpaceC), _u64p, ctypes.c_uint64, P(Breakdown), _u32p]
        _lib.or_stage_layers.argtypes = [P(Model), P(Cfg), ctypes.c_uint32]
        _lib.or_stage_layers.restype = ctypes.c_uint32
        _lib.or_estimate_stage.argtypes = [P(Model), P(Cfg), ctypes.c_uint32, P(Breakdown)]
        _lib.or_estimate_max.argtypes = [P(Model), P(Cfg), P(Breakdown), _u32p]
        _lib.or_digest.argtypes = [P(SpaceC), ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                   _u64p]
    return _lib


def _model(shape) -> Model:
    return Model(*[int(x) for x in shape])


def _scalar(fn, shape, *args):
    out = ctypes.c_uint64()
    st = fn(ctypes.byref(_model(shape)), *args, ctypes.byref(out))
    if st:
        raise OracleError(st, fn.__name__)
    return out.value


def attention_params(shape):
    return _scalar(lib().or_attention_params, shape)


def ffn_params(shape):
    return _scalar(lib().or_ffn_params, shape)


def total_params(shape):
    return _scalar(lib().or_total_params, shape)


def stage0_params(shape, t, p, L0):
    return _scalar(lib().or_stage0_params, shape, t, p, L0)


def activation_per_layer(shape, s, b):
    return _scalar(lib().or_activation_per_layer, shape, s, b)


def make_cfg(d, t, p, c, b, s, gbs=0, L0=0, rc=0, dopt=1, uneven=0, zero=0, sp_off=0, vpp=0, wb=0, gb=0,
             ob=0) -> Cfg:
    return Cfg(d, t, p, c, b, s, gbs, L0, rc, dopt, uneven, zero, sp_off, vpp, wb, gb, ob)


def first_stage_layers(shape, **cfg):
    return lib().or_first_stage_layers(ctypes.byref(_model(shape)), ctypes.byref(make_cfg(**cfg)))


def estimate(shape, **cfg) -> dict:
    """Eq.18 terms for one config; raises OracleError on a precondition failure."""
    out = Breakdown()
    st = lib().or_estimate(ctypes.byref(_model(shape)), ctypes.byref(make_cfg(**cfg)),
                           ctypes.byref(out))
    if st:
        raise OracleError(st, str(cfg))
    return {k: getattr(out, k) for k in TERMS}


def estimate_status(shape, **cfg) -> int:
    out = Breakdown()
    return lib().or_estimate(ctypes.byref(_model(shape)), ctypes.byref(make_cfg(**cfg)),
                             ctypes.byref(out))


def stage_layers(shape, stage, **cfg) -> int:
    return lib().or_stage_layers(ctypes.byref(_model(shape)), ctypes.byref(make_cfg(**cfg)), stage)


def estimate_stage(shape, stage, **cfg) -> dict:
    """NEXT-1: the six terms of pipeline stage `stage` (Eq.6-9, 1F1B occupancy)."""
    out = Breakdown()
    st = lib().or_estimate_stage(ctypes.byref(_model(shape)), ctypes.byref(make_cfg(**cfg)), stage,
                                 ctypes.byref(out))
    if st:
        raise OracleError(st, f"stage {stage} {cfg}")
    return {k: getattr(out, k) for k in TERMS}


def estimate_max(shape, **cfg):
    """NEXT-1: (terms of the stage with the largest total, that stage)."""
    out, stage = Breakdown(), ctypes.c_uint32()
    st = lib().or_estimate_max(ctypes.byref(_model(shape)), ctypes.byref(make_cfg(**cfg)), ctypes.byref(out),
                               ctypes.byref(stage))
    if st:
        raise OracleError(st, str(cfg))
    return {k: getattr(out, k) for k in TERMS}, stage.value


def cap_mask(total, cap_bytes, num=4, den=5) -> int:
    caps = (ctypes.c_uint64 * max(1, len(cap_bytes)))(*cap_bytes)
    return lib().or_cap_mask(total, caps, len(cap_bytes), num, den)


class _SpaceHolder:
    """Keeps the ctypes arrays alive for the lifetime of the struct."""

    def __init__(self, sp):
        self.models = (Model * len(sp.models))(*[_model(m) for m in sp.models])
        self.world = (ctypes.c_uint32 * len(sp.world))(*sp.world)
        cb = sp.cap_bytes
        self.caps = (ctypes.c_uint64 * max(1, len(cb)))(*cb)
        self.mbs = (ctypes.c_uint32 * len(sp.mbs))(*sp.mbs)
        self.seq = (ctypes.c_uint32 * len(sp.seq))(*sp.seq)
        self.c = SpaceC(self.models, len(sp.models), self.world, len(sp.world), self.caps, len(cb),
                        sp.gpus_per_node, self.mbs, len(sp.mbs), self.seq, len(sp.seq),
                        sp.rc_mask, sp.do_mask, sp.uneven, getattr(sp, "stage_max", 0), sp.gbs, sp.max_t, sp.max_c,
                        sp.max_p, sp.thr_num, sp.thr_den, getattr(sp, "zero_stage", 0),
                        getattr(sp, "sp_off", 0), getattr(sp, "vpp", 0), getattr(sp, "wb", 0), getattr(sp, "gb", 0),
                        getattr(sp, "ob", 0))


def space_size(sp) -> int:
    h = _SpaceHolder(sp)
    n = ctypes.c_uint64()
    st = lib().or_space_size(ctypes.byref(h.c), ctypes.byref(n))
    if st:
        raise OracleError(st, "space_size")
    return n.value


def decode(sp, index):
    h = _SpaceHolder(sp)
    mid, world, cfg = ctypes.c_uint32(), ctypes.c_uint32(), Cfg()
    st = lib().or_decode(ctypes.byref(h.c), index, ctypes.byref(mid), ctypes.byref(world),
                         ctypes.byref(cfg))
    if st:
        raise OracleError(st, f"decode {index}")
    return mid.value, world.value, {k: getattr(cfg, k) for k in
                                    ("d", "t", "p", "c", "b", "s", "gbs", "rc", "dopt")}


def sweep(sp, begin=0, end=0, rows=True, threads=None, max_rows=None):
    """Survivors of [begin, end) in ascending index order.

    Returns (idx_mask uint64[n], rows uint64[n, 7] or None, count, cap_counts)."""
    h = _SpaceHolder(sp)
    threads = threads or 1
    count = ctypes.c_uint64()
    cc = (ctypes.c_uint64 * 8)()
    if rows:
        if max_rows is None:
            n_all = (end or space_size(sp)) - begin
            max_rows = max(1, n_all)
        idx = np.zeros(max_rows, dtype=np.uint64)
        rw = np.zeros((max_rows, 7), dtype=np.uint64)
        st = lib().or_sweep(ctypes.byref(h.c), begin, end, idx.ctypes.data_as(_u64p),
                            rw.ctypes.data_as(ctypes.POINTER(Breakdown)), max_rows,
                            ctypes.byref(count), cc, threads)
    else:
        st = lib().or_sweep(ctypes.byref(h.c), begin, end, None, None, 0, ctypes.byref(count), cc,
                            threads)
    if st:
        raise OracleError(st, "sweep")
    n = count.value
    caps = [cc[i] for i in range(len(sp.cap_bytes))]
    if rows:
        return idx[:n].copy(), rw[:n].copy(), n, caps
    return None, None, n, caps


def points(sp, indices):
    """Records (rows uint64[n, 7], masks uint32[n]) of the configurations at the
    given indices, evaluated one by one in a single canonical walk."""
    h = _SpaceHolder(sp)
    order = np.argsort(np.asarray(indices, dtype=np.uint64), kind="stable")
    pts = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64)[order])
    rows = np.zeros((len(pts), 7), dtype=np.uint64)
    masks = np.zeros(len(pts), dtype=np.uint32)
    st = lib().or_points(ctypes.byref(h.c), pts.ctypes.data_as(_u64p), len(pts),
                         rows.ctypes.data_as(ctypes.POINTER(Breakdown)), masks.ctypes.data_as(_u32p))
    if st:
        raise OracleError(st, "points")
    inv = np.empty_like(order)
    inv[order] = np.arange(len(order))
    return rows[inv], masks[inv]


DIGEST_WORDS = 11  # count, 8 per-capacity counts, index digest, record digest


def digest(sp, begin=0, end=0, chunk=1 << 28, threads=None):
    """Per chunk of [begin, end): (count, cap_counts[8], index digest, record
    digest) as a uint64 array (n_chunks, 11); the digest definition is in
    me_oracle.h (or_digest).  Test infrastructure for whole-chunk parity."""
    h = _SpaceHolder(sp)
    end = end or space_size(sp)
    n_chunks = max(0, -(-(end - begin) // chunk))
    out = np.zeros((max(1, n_chunks), DIGEST_WORDS), dtype=np.uint64)
    st = lib().or_digest(ctypes.byref(h.c), begin, end, chunk, threads or default_threads(),
                         out.ctypes.data_as(_u64p))
    if st:
        raise OracleError(st, "digest")
    return out[:n_chunks]


def digest_of_rows(idx_mask, rows):
    """The same digest from explicit survivor rows (numpy, for the pins)."""
    C, M = 0x9E3779B97F4A7C15, 0xD1B54A32D192ED03
    W = (1 << 64) - 1

    def mix(x):
        x ^= x >> 30
        x = (x * 0xBF58476D1CE4E5B9) & W
        x ^= x >> 27
        x = (x * 0x94D049BB133111EB) & W
        x ^= x >> 31
        return x

    di = dr = 0
    pw = 1
    for j in range(len(idx_mask)):
        r = [int(idx_mask[j])] + [int(x) for x in rows[j]]
        gi = mix((r[0] + C) & W)
        gr = C
        for v in r:
            gr = mix(gr ^ v)
        di = (di + gi * pw) & W
        dr = (dr + gr * pw) & W
        pw = (pw * M) & W
    return di, dr


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


# ---------------------------------------------------------------------------
# NEXT-2 planner reference (test infrastructure): schedule statistics, the
# 3-class colouring and the survey's ranking, restated in plain Python over
# the oracle's own enumeration and totals.  Small spaces only.
# ---------------------------------------------------------------------------

def enumerate_configs(sp):
    """The canonical enumeration as plain nested loops, in index
    order: yields (index, model_id, N, dict(d, t, c, p, b, s, rc, dopt))."""
    idx = 0
    for mid, (h, f, L, a, k, v) in enumerate(sp.models):
        for N in sp.world:
            for t in range(1, N + 1):
                if N % t:
                    continue
                for c in range(1, N // t + 1):
                    if (N // t) % c:
                        continue
                    for p in range(1, N // t // c + 1):
                        if (N // t // c) % p:
                            continue
                        d = N // (t * c * p)
                        if k % t or v % t or f % t or p > L or (not sp.uneven and L % p):
                            continue
                        if sp.vpp >= 2 and (p < 2 or L % (p * sp.vpp)):
                            continue
                        if (sp.max_t and t > sp.max_t) or (sp.max_c and c > sp.max_c) or (sp.max_p and p > sp.max_p):
                            continue
                        if sp.gpus_per_node and t > sp.gpus_per_node:
                            continue
                        for b in sp.mbs:
                            for s in sp.seq:
                                if s % c or (sp.gbs and sp.gbs % (d * b)):
                                    continue
                                if sp.gbs and sp.vpp >= 2 and (sp.gbs // (d * b)) % p:
                                    continue
                                for rc in (0, 1):
                                    if not (sp.rc_mask >> rc) & 1:
                                        continue
                                    for dopt in (0, 1):
                                        if not (sp.do_mask >> dopt) & 1:
                                            continue
                                        yield idx, mid, N, dict(d=d, t=t, c=c, p=p, b=b, s=s, rc=rc, dopt=dopt)
                                        idx += 1


def schedule_stats(gbs, d, b, p):
    """SPEC S:226-244 / P:566-567: microbatches m = GBS/(d b), the 1F1B pipeline
    bubble fraction (p - 1)/m as (numerator, denominator), and the per-stage
    peak in-flight microbatches min(m, p - i)."""
    if gbs % (d * b):
        raise ValueError("(d b) must divide the global batch")
    m = gbs // (d * b)
    return m, (p - 1, m), [min(m, p - i) for i in range(p)]


def feasibility_class(total, cap_bytes, num=4, den=5):
    """Caption P:420 / SPEC S:325-331: 0 green (total <= num/den of the
    capacity, ties green, R3), 1 yellow (<= the capacity), 2 red."""
    if total * den <= cap_bytes * num:
        return 0
    return 1 if total <= cap_bytes else 2


def rank(sp, cap_bytes, gpus_per_node=0, k=1, num=4, den=5):
    """Per (model, N) segment, the k best configurations of the space by the
    survey's key: (1) class green <
    yellow < red, (2) t <= gpus_per_node before t > gpus_per_node (P:48-49,
    P:564), (3) ascending t*c*p, (4) descending b,
    (5) ascending p (bubble), (6) ascending c, (7) ascending t; then
    recompute off first and the smallest index.  Returns {segment: [(index,
    class, (t, c, p, b))...]} over every configuration of the space (red
    included), segment = model_id * len(world) + world position."""
    import dataclasses
    everything = dataclasses.replace(sp, caps_gb=[], caps_bytes=[(1 << 64) - 1], thr_num=1, thr_den=1)
    idx, rows, n, _ = sweep(everything, threads=default_threads())
    totals = {int(i) & ((1 << 56) - 1): int(r[6]) for i, r in zip(idx, rows)}
    segs = {}
    for i, mid, N, cfg in enumerate_configs(sp):
        cls = feasibility_class(totals[i], cap_bytes, num, den)
        node = 1 if gpus_per_node and cfg["t"] > gpus_per_node else 0
        key = (cls, node, cfg["t"] * cfg["c"] * cfg["p"], -cfg["b"], cfg["p"], cfg["c"], cfg["t"], cfg["rc"], i)
        segs.setdefault(mid * len(sp.world) + sp.world.index(N), []).append(
            (key, (i, cls, (cfg["t"], cfg["c"], cfg["p"], cfg["b"]))))
    return {s: [x for _, x in sorted(v)[:k]] for s, v in segs.items()}
