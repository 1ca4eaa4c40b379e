"""me-b200: exact 4D-parallel LLM memory-estimator sweeps on NVIDIA B200.

Thin Python binding over libme.so (include/me.h); names follow the C ABI.
PyTorch supplies device memory (its caching allocator, through the ABI's
allocator callbacks), streams and process groups -- nothing else.  Every
estimator step runs in the library's sm_100a kernels; importing this package
fails loudly when the library is missing (there is no CPU fallback).

Paper: Fujii, Watanabe, Yokota, "Accelerating Large Language Model Training
with 4D Parallelism and Memory Consumption Estimator", arXiv 2411.06465
(estimator: Eq.1-18; 80% rule: P:27).
"""
from __future__ import annotations

import ctypes
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _abi
from ._abi import (ME_N_COLS, ME_OUT_COUNT, ME_OUT_FULL, ME_OUT_INDEX, ME_OUT_RECORDS, ME_PART_CYCLIC, ME_PART_EVEN,
                   MEError, check, lib, me_breakdown,
                   me_cfg_range, me_cluster, me_model, me_model_range, me_parallel, me_sweep_opts, me_threshold)

lib()  # fail at import time when libme.so is absent

TERMS = ("params", "grads", "optim", "act_layers", "act_embed", "act_head", "total")
COLUMNS = ("index_mask",) + TERMS
GIB = 1 << 30


def version() -> str:
    return lib().me_version().decode()


def _parallel(d, t, p, c, b, s, gbs=0, L0=0, rc=0, dopt=1, uneven=0, zero=0, sp_off=0, vpp=0, wb=0, gb=0,
              ob=0) -> me_parallel:
    return me_parallel(d, t, p, c, b, s, gbs, L0, rc, dopt, uneven, zero, sp_off, vpp, wb, gb, ob)


def me_estimate(shape, **cfg) -> Dict[str, int]:
    """Eq.18 terms of one configuration on the current CUDA device.
    cfg keys: d, t, p, c, b, s, gbs, L0, rc, dopt, uneven."""
    out = me_breakdown()
    check(lib().me_estimate(ctypes.byref(me_model(*shape)), ctypes.byref(_parallel(**cfg)), ctypes.byref(out)),
          "me_estimate")
    return {k: getattr(out, k) for k in TERMS}


STAGE_ARGMAX = 0xFFFFFFFF


def me_estimate_stage(shape, stage, **cfg):
    """NEXT-1: terms of pipeline stage `stage` (or STAGE_ARGMAX: the largest);
    returns (terms, stage index)."""
    out, which = me_breakdown(), ctypes.c_uint32()
    check(lib().me_estimate_stage(ctypes.byref(me_model(*shape)), ctypes.byref(_parallel(**cfg)), stage,
                                  ctypes.byref(out), ctypes.byref(which)), "me_estimate_stage")
    return {k: getattr(out, k) for k in TERMS}, which.value


def me_estimate_batch(shapes: Sequence, ids, cfgs: Sequence[dict], caps_bytes=(), thr=(4, 5), stream=None):
    """Batched single estimates.  Returns (rows uint64[n, 7], cap_mask uint8[n], status uint8[n])."""
    n = len(cfgs)
    models = (me_model * len(shapes))(*[me_model(*s) for s in shapes])
    ida = np.ascontiguousarray(np.asarray(ids, dtype=np.uint32)) if ids is not None else None
    arr = (me_parallel * max(1, n))(*[_parallel(**c) for c in cfgs])
    caps = np.ascontiguousarray(np.asarray(caps_bytes, dtype=np.uint64))
    rows = np.zeros((n, 7), dtype=np.uint64)
    mask = np.zeros(n, dtype=np.uint8)
    status = np.zeros(n, dtype=np.uint8)
    check(lib().me_estimate_batch(models, len(shapes), ida.ctypes.data if ida is not None else None, arr, n,
                                  caps.ctypes.data if len(caps) else None, len(caps), me_threshold(*thr),
                                  rows.ctypes.data, mask.ctypes.data, status.ctypes.data, stream),
          "me_estimate_batch")
    return rows, mask, status


class _SpaceC:
    """C structs for a space description (any object with the attributes of
    me_inputs.Space: models, world, caps_gb or cap_bytes, mbs, seq, masks...)."""

    def __init__(self, sp):
        self.models = (me_model * len(sp.models))(*[me_model(*m) for m in sp.models])
        self.world = (ctypes.c_uint32 * len(sp.world))(*sp.world)
        cb = list(sp.cap_bytes)
        self.caps = (ctypes.c_uint64 * max(1, len(cb)))(*cb)
        self.mbs = (ctypes.c_uint32 * len(sp.mbs))(*sp.mbs)
        self.seq = (ctypes.c_uint32 * len(sp.seq))(*sp.seq)
        self.mr = me_model_range(self.models, len(sp.models))
        self.cl = me_cluster(self.world, len(sp.world), self.caps, len(cb), sp.gpus_per_node)
        self.cr = me_cfg_range(self.mbs, len(sp.mbs), self.seq, len(sp.seq), sp.rc_mask, sp.do_mask, sp.uneven,
                               getattr(sp, "stage_max", 0),
                               sp.gbs, sp.max_t, sp.max_c, sp.max_p, getattr(sp, "zero_stage", 0),
                               getattr(sp, "sp_off", 0), getattr(sp, "vpp", 0), getattr(sp, "wb", 0),
                               getattr(sp, "gb", 0), getattr(sp, "ob", 0))
        self.thr = me_threshold(sp.thr_num, sp.thr_den)
        self.n_cap = len(cb)


def me_space_size(sp) -> int:
    c = _SpaceC(sp)
    n = ctypes.c_uint64()
    check(lib().me_space_size(ctypes.byref(c.mr), ctypes.byref(c.cl), ctypes.byref(c.cr), ctypes.byref(n)),
          "me_space_size")
    return n.value


def me_decode(sp, index: int):
    c = _SpaceC(sp)
    mid, world, out = ctypes.c_uint32(), ctypes.c_uint32(), me_parallel()
    check(lib().me_decode(ctypes.byref(c.mr), ctypes.byref(c.cl), ctypes.byref(c.cr), index, ctypes.byref(mid),
                          ctypes.byref(world), ctypes.byref(out)), "me_decode")
    cfg = dict(d=out.dp, t=out.tp, p=out.pp, c=out.cp, b=out.mbs, s=out.seq, gbs=out.gbs, rc=out.recompute,
               dopt=out.dist_opt)
    for k in ("sp_off", "vpp"):
        if getattr(out, k):
            cfg[k] = getattr(out, k)
    return mid.value, world.value, cfg


class TorchAllocator:
    """me_alloc_fn / me_free_fn backed by PyTorch's caching allocator.  Keeps
    the tensors alive by pointer so results can be handed out as tensors."""

    def __init__(self, device: int):
        import torch
        self.torch = torch
        self.device = device
        self.live: Dict[int, "torch.Tensor"] = {}
        self.c_alloc = _abi.me_alloc_fn(self._alloc)
        self.c_free = _abi.me_free_fn(self._free)

    def _alloc(self, nbytes, stream, ctx):
        torch = self.torch
        try:
            s = torch.cuda.ExternalStream(stream, device=self.device) if stream else torch.cuda.default_stream(
                self.device)
            with torch.cuda.device(self.device), torch.cuda.stream(s):
                t = torch.empty((nbytes + 7) // 8, dtype=torch.int64, device=f"cuda:{self.device}")
        except Exception:
            return None
        ptr = t.data_ptr()
        self.live[ptr] = t
        return ptr

    def _free(self, ptr, stream, ctx):
        self.live.pop(ptr, None)

    def tensor(self, ptr: int, n: int):
        t = self.live.get(ptr)
        return None if t is None else t[:n]


class Result:
    def __init__(self, handle, plan: "Plan", mode: int, n_cap: int, user_cols=None):
        self.h = ctypes.c_void_p(handle)
        self.plan = plan
        self.mode = mode
        self.n_cap = n_cap
        self.user_cols = user_cols

    def counts(self):
        lo, gl, off = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        check(lib().me_result_counts(self.h, ctypes.byref(lo), ctypes.byref(gl), ctypes.byref(off)),
              "me_result_counts")
        return lo.value, gl.value, off.value

    @property
    def count(self) -> int:
        return self.counts()[1]

    def cap_counts(self) -> List[int]:
        a = (ctypes.c_uint64 * 8)()
        check(lib().me_result_cap_counts(self.h, a), "me_result_cap_counts")
        return [a[i] for i in range(self.n_cap)]

    def status(self) -> int:
        return lib().me_result_status(self.h)

    def wait(self):
        check(lib().me_result_wait(self.h), "me_result_wait")

    def timing(self):
        a = (ctypes.c_float * 4)()
        check(lib().me_result_timing(self.h, a), "me_result_timing")
        return list(a)

    def columns(self):
        """Device columns as torch int64 tensors (u64 bit patterns), or None;
        RECORDS: column 0 is an (n, 8) tensor of me_record rows."""
        ptrs = (ctypes.c_void_p * ME_N_COLS)()
        n = ctypes.c_uint64()
        check(lib().me_result_columns(self.h, ptrs, ctypes.byref(n)), "me_result_columns")
        wd = 8 if self.mode == ME_OUT_RECORDS else 1
        out = []
        for j in range(ME_N_COLS):
            p = ptrs[j]
            if not p:
                out.append(None)
                continue
            t = self.plan.alloc.tensor(p, n.value * wd) if self.plan.alloc else None
            if t is None and self.user_cols is not None:
                t = self.user_cols[j].reshape(-1)[:n.value * wd]
            out.append(t.view(-1, 8) if wd == 8 and t is not None else t)
        return out, n.value

    def to_host(self, first: int = 0, n: Optional[int] = None) -> Dict[str, np.ndarray]:
        ptrs = (ctypes.c_void_p * ME_N_COLS)()
        rows = ctypes.c_uint64()
        check(lib().me_result_columns(self.h, ptrs, ctypes.byref(rows)), "me_result_columns")
        if n is None:
            n = rows.value - first
        if self.mode == ME_OUT_RECORDS:  # one (n, 8) array of records, returned as its columns
            rec = np.zeros((n, 8), dtype=np.uint64)
            hp = (ctypes.c_void_p * ME_N_COLS)(*([rec.ctypes.data] + [None] * (ME_N_COLS - 1)))
            check(lib().me_result_copy_to_host(self.h, first, n, hp), "me_result_copy_to_host")
            return dict(zip(COLUMNS, (rec[:, j] for j in range(8))))
        ncol = 8 if self.mode == ME_OUT_FULL else (1 if self.mode == ME_OUT_INDEX else 0)
        arrays = [np.zeros(n, dtype=np.uint64) for _ in range(ncol)]
        hp = (ctypes.c_void_p * ME_N_COLS)(*([a.ctypes.data for a in arrays] + [None] * (ME_N_COLS - ncol)))
        check(lib().me_result_copy_to_host(self.h, first, n, hp), "me_result_copy_to_host")
        return dict(zip(COLUMNS, arrays))

    def rank(self, green_cap: int = 0, yellow_cap: Optional[int] = None, gpus_per_node: int = 0, k: int = 1):
        """NEXT-2 (me_result_rank): per (model, N) segment the k best rows by the
        survey's key; a list per segment of dicts (index, class 0/1/2 = green /
        yellow / red, t, c, p, d, b, s, rc, dopt, microbatches, bubble as
        (p - 1, m)), rows past a segment's result rows omitted."""
        n_seg = len(self.plan.c.models) * len(self.plan.c.world)
        out = (_abi.me_rank_row * (n_seg * k))()
        o = _abi.me_rank_opts(green_cap, _abi.ME_RANK_NONE if yellow_cap is None else yellow_cap, gpus_per_node, k)
        check(lib().me_result_rank(self.h, ctypes.byref(o), out), "me_result_rank")
        segs = []
        for s_ in range(n_seg):
            rows = []
            for q in range(k):
                x = out[s_ * k + q]
                if x.index == 0xFFFFFFFFFFFFFFFF:
                    break
                c = x.cfg
                rows.append(dict(index=x.index, key=x.key, cls=x.cls, model_id=x.model_id, world=x.world_size,
                                 t=c.tp, c=c.cp, p=c.pp, d=c.dp, b=c.mbs, s=c.seq, rc=c.recompute, dopt=c.dist_opt,
                                 microbatches=x.microbatches, bubble=(x.bubble_num, x.bubble_den)))
            segs.append(rows)
        return segs

    def digest(self):
        """(index digest, record digest) of the result's rows (me_result_digest;
        collective for a sharded comm result)."""
        a = (ctypes.c_uint64 * 2)()
        check(lib().me_result_digest(self.h, a), "me_result_digest")
        return a[0], a[1]

    def free(self):
        if self.h:
            lib().me_result_free(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Comm:
    """NCCL communicator bootstrapped through torch.distributed (any backend)."""

    def __init__(self, device: int):
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        uid = (ctypes.c_uint8 * 128)()
        if rank == 0:
            check(lib().me_comm_unique_id(uid), "me_comm_unique_id")
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        uid = (ctypes.c_uint8 * 128)(*obj[0])
        h = ctypes.c_void_p()
        check(lib().me_comm_init(uid, rank, world, device, ctypes.byref(h)), "me_comm_init")
        self.h = h
        self.rank, self.world = rank, world

    def check(self):
        """raise if NCCL recorded an asynchronous error on this communicator"""
        check(lib().me_comm_check(self.h), "me_comm_check")

    def destroy(self):
        if self.h:
            lib().me_comm_destroy(self.h)
            self.h = ctypes.c_void_p()


class Plan:
    """Enumeration tables of a space resident on one GPU (me_plan_create)."""

    def __init__(self, sp, device: int = 0, stream=None, use_torch_alloc: bool = True):
        self.c = _SpaceC(sp)
        self.device = device
        self.stream = stream
        self.alloc = TorchAllocator(device) if use_torch_alloc else None
        h = ctypes.c_void_p()
        a = self.alloc.c_alloc if self.alloc else _abi.me_alloc_fn()
        f = self.alloc.c_free if self.alloc else _abi.me_free_fn()
        check(lib().me_plan_create(ctypes.byref(self.c.mr), ctypes.byref(self.c.cl), ctypes.byref(self.c.cr), self.c.thr,
                                   device, stream, a, f, None, ctypes.byref(h)), "me_plan_create")
        self.h = h
        n = ctypes.c_uint64()
        check(lib().me_plan_size(self.h, ctypes.byref(n)), "me_plan_size")
        self.size = n.value
        check(lib().me_plan_table_bytes(self.h, ctypes.byref(n)), "me_plan_table_bytes")
        self.table_bytes = n.value

    def sweep(self, begin: int = 0, end: int = 0, mode: int = ME_OUT_FULL, out_cols=None, comm: Optional[Comm] = None,
              gather: bool = False, partition: int = ME_PART_EVEN) -> Result:
        """me_plan_sweep.  out_cols: optional list of torch int64 device tensors
        (8 for FULL, 1 for INDEX) of equal length = capacity; RECORDS: one
        tensor of 8 * capacity elements.  partition = ME_PART_CYCLIC: this call
        is one block of a cyclic deal (see cyclic_blocks / result_join)."""
        cols_arr = None
        cap = 0
        if out_cols is not None:
            cols_arr = (ctypes.c_void_p * ME_N_COLS)(*([t.data_ptr() for t in out_cols] +
                                                       [None] * (ME_N_COLS - len(out_cols))))
            cap = min(t.numel() for t in out_cols) // (8 if mode == ME_OUT_RECORDS else 1)
        o = me_sweep_opts(begin, end, mode, self.device, self.stream, _abi.me_alloc_fn(), _abi.me_free_fn(), None,
                          comm.h if comm else None, 1 if gather else 0, 0, cols_arr, cap, partition, 0)
        h = ctypes.c_void_p()
        check(lib().me_plan_sweep(self.h, ctypes.byref(o), ctypes.byref(h)), "me_plan_sweep")
        return Result(h.value, self, mode, self.c.n_cap, user_cols=out_cols)

    def free(self):
        if self.h:
            lib().me_plan_free(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def me_sweep(sp, begin: int = 0, end: int = 0, mode: int = ME_OUT_FULL, device: int = 0, stream=None,
             comm: Optional[Comm] = None, gather: bool = False) -> Result:
    """One-shot sweep (plan + sweep); the plan lives as long as the result."""
    plan = Plan(sp, device=device, stream=stream)
    r = plan.sweep(begin, end, mode, comm=comm, gather=gather)
    r._plan_ref = plan
    return r


def cyclic_blocks(begin: int, end: int, block: int, rank: int, nranks: int):
    """a8 cyclic partition (me_cyclic_block): this rank's blocks [(lo, hi)] in
    order (block q of [begin, end) belongs to rank q mod nranks) and the total
    number of blocks."""
    out, k = [], 0
    lo, hi, nb = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    while True:
        st = lib().me_cyclic_block(begin, end, block, rank, nranks, k, ctypes.byref(lo), ctypes.byref(hi),
                                   ctypes.byref(nb))
        if st == _abi.ME_ERANGE:
            return out, nb.value
        check(st, "me_cyclic_block")
        out.append((lo.value, hi.value))
        k += 1


def result_join(results: Sequence["Result"], n_blocks: int, comm: "Comm"):
    """a8 deferred join (me_result_join): one NCCL allgather of every block's
    counts and the exclusive scan on the device; collective over comm."""
    arr = (ctypes.c_void_p * max(1, len(results)))(*[r.h.value for r in results])
    check(lib().me_result_join(arr, len(results), n_blocks, comm.h), "me_result_join")


def digest_merge(counts, digests):
    """me_digest_merge: the digest of consecutive pieces (counts[i] rows,
    digests[i] = (index, record)) of one result.  Host-only."""
    n = len(counts)
    c = (ctypes.c_uint64 * max(1, n))(*[int(x) for x in counts])
    d = (ctypes.c_uint64 * max(2, 2 * n))(*[int(x) for pair in digests for x in pair])
    out = (ctypes.c_uint64 * 2)()
    check(lib().me_digest_merge(n, c, d, out), "me_digest_merge")
    return out[0], out[1]
