"""ctypes mirror of include/me.h.  Argument marshalling only: every step of the
estimator runs inside libme.so (CUDA kernels for sm_100a).  There is no Python
or CPU fallback; loading fails loudly when the library is missing."""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
# ME_CHECKED=1 loads the build with device-side bounds assertions
# (libme_checked.so, paper_2411_06465_b200/build.py --checked); tests only
LIB_PATH = PKG / ("libme_checked.so" if os.environ.get("ME_CHECKED") == "1" else "libme.so")

ME_OK, ME_EINVAL, ME_EDIV, ME_EOVERFLOW, ME_ENOMEM, ME_ECUDA, ME_ENCCL, ME_ERANGE = range(8)
ME_OUT_COUNT, ME_OUT_INDEX, ME_OUT_FULL, ME_OUT_RECORDS = 0, 1, 2, 3
ME_PART_EVEN, ME_PART_CYCLIC = 0, 1
ME_N_COLS = 8

u8, u32, u64 = ctypes.c_uint8, ctypes.c_uint32, ctypes.c_uint64
P = ctypes.POINTER


class me_model(ctypes.Structure):
    _fields_ = [(n, u32) for n in ("hidden", "ffn_hidden", "layers", "heads", "kv_heads", "vocab")]


class me_parallel(ctypes.Structure):
    _fields_ = [(n, u32) for n in ("dp", "tp", "pp", "cp", "mbs", "seq", "gbs", "first_stage_layers")] + [
        ("recompute", u8), ("dist_opt", u8), ("allow_uneven_pp", u8), ("zero_stage", u8)] + [
        (n, u8) for n in ("sp_off", "vpp", "w_bytes", "g_bytes", "o_bytes", "_pad0", "_pad1", "_pad2")]


class me_breakdown(ctypes.Structure):
    _fields_ = [(n, u64) for n in ("params", "grads", "optim", "act_layers", "act_embed", "act_head", "total")]


class me_threshold(ctypes.Structure):
    _fields_ = [("num", u32), ("den", u32)]


class me_model_range(ctypes.Structure):
    _fields_ = [("models", P(me_model)), ("n_models", u32)]


class me_cluster(ctypes.Structure):
    _fields_ = [("world_sizes", P(u32)), ("n_world", u32), ("capacity_bytes", P(u64)), ("n_cap", u32),
                ("gpus_per_node", u32)]


class me_cfg_range(ctypes.Structure):
    _fields_ = [("mbs", P(u32)), ("n_mbs", u32), ("seq", P(u32)), ("n_seq", u32),
                ("recompute_mask", u8), ("dist_opt_mask", u8), ("allow_uneven_pp", u8), ("stage_policy", u8),
                ("gbs", u32), ("max_tp", u32), ("max_cp", u32), ("max_pp", u32), ("zero_stage", u32)] + [
        (n, u8) for n in ("sp_off", "vpp", "w_bytes", "g_bytes", "o_bytes", "_pad0", "_pad1", "_pad2")]


me_alloc_fn = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
me_free_fn = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class me_sweep_opts(ctypes.Structure):
    _fields_ = [("begin", u64), ("end", u64), ("mode", ctypes.c_int), ("device", ctypes.c_int),
                ("stream", ctypes.c_void_p), ("alloc", me_alloc_fn), ("free", me_free_fn),
                ("alloc_ctx", ctypes.c_void_p), ("comm", ctypes.c_void_p), ("gather", u32), ("_pad", u32),
                ("out_cols", P(ctypes.c_void_p)), ("out_capacity", u64), ("partition", ctypes.c_int), ("_pad2", u32)]


ME_RANK_NONE = 0xFFFFFFFF


class me_rank_opts(ctypes.Structure):
    _fields_ = [("green_cap", u32), ("yellow_cap", u32), ("gpus_per_node", u32), ("k", u32)]


class me_rank_row(ctypes.Structure):
    _fields_ = [("index", u64), ("key", u64), ("model_id", u32), ("world_size", u32), ("cfg", me_parallel),
                ("cls", u32), ("microbatches", u32), ("bubble_num", u32), ("bubble_den", u32), ("_pad", u32)]


class MEError(RuntimeError):
    def __init__(self, status: int, call: str, detail: str = ""):
        super().__init__(f"{call}: status {status} ({strerror(status)}) {detail}")
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: build it with paper_2411_06465_b200.build "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(str(LIB_PATH))
        sigs = {
            "me_estimate": ([P(me_model), P(me_parallel), P(me_breakdown)], ctypes.c_int),
            "me_estimate_stage": ([P(me_model), P(me_parallel), u32, P(me_breakdown), P(u32)], ctypes.c_int),
            "me_estimate_batch": ([ctypes.c_void_p, u32, ctypes.c_void_p, ctypes.c_void_p, u64, ctypes.c_void_p,
                                   u32, me_threshold, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p], ctypes.c_int),
            "me_space_size": ([P(me_model_range), P(me_cluster), P(me_cfg_range), P(u64)], ctypes.c_int),
            "me_decode": ([P(me_model_range), P(me_cluster), P(me_cfg_range), u64, P(u32), P(u32),
                           P(me_parallel)], ctypes.c_int),
            "me_plan_create": ([P(me_model_range), P(me_cluster), P(me_cfg_range), me_threshold, ctypes.c_int,
                                ctypes.c_void_p, me_alloc_fn, me_free_fn, ctypes.c_void_p,
                                P(ctypes.c_void_p)], ctypes.c_int),
            "me_plan_size": ([ctypes.c_void_p, P(u64)], ctypes.c_int),
            "me_plan_table_bytes": ([ctypes.c_void_p, P(u64)], ctypes.c_int),
            "me_plan_sweep": ([ctypes.c_void_p, P(me_sweep_opts), P(ctypes.c_void_p)], ctypes.c_int),
            "me_plan_free": ([ctypes.c_void_p], None),
            "me_sweep": ([P(me_model_range), P(me_cluster), P(me_cfg_range), me_threshold, P(me_sweep_opts),
                          P(ctypes.c_void_p)], ctypes.c_int),
            "me_result_counts": ([ctypes.c_void_p, P(u64), P(u64), P(u64)], ctypes.c_int),
            "me_result_cap_counts": ([ctypes.c_void_p, P(u64)], ctypes.c_int),
            "me_result_columns": ([ctypes.c_void_p, P(ctypes.c_void_p), P(u64)], ctypes.c_int),
            "me_result_copy_to_host": ([ctypes.c_void_p, u64, u64, P(ctypes.c_void_p)], ctypes.c_int),
            "me_result_status": ([ctypes.c_void_p], ctypes.c_int),
            "me_result_wait": ([ctypes.c_void_p], ctypes.c_int),
            "me_result_timing": ([ctypes.c_void_p, P(ctypes.c_float)], ctypes.c_int),
            "me_result_free": ([ctypes.c_void_p], None),
            "me_result_rank": ([ctypes.c_void_p, P(me_rank_opts), P(me_rank_row)], ctypes.c_int),
            "me_result_digest": ([ctypes.c_void_p, P(u64)], ctypes.c_int),
            "me_digest_merge": ([u64, P(u64), P(u64), P(u64)], ctypes.c_int),
            "me_comm_check": ([ctypes.c_void_p], ctypes.c_int),
            "me_cyclic_block": ([u64, u64, u64, ctypes.c_int, ctypes.c_int, u64, P(u64), P(u64), P(u64)], ctypes.c_int),
            "me_result_join": ([P(ctypes.c_void_p), u32, u64, ctypes.c_void_p], ctypes.c_int),
            "me_partition": ([u64, u64, ctypes.c_int, ctypes.c_int, P(u64), P(u64)], ctypes.c_int),
            "me_join_counts": ([P(u64), ctypes.c_int, u32, u32, ctypes.c_int, P(u64), P(u64), P(u64)], ctypes.c_int),
            "me_comm_unique_id": ([P(u8)], ctypes.c_int),
            "me_comm_init": ([P(u8), ctypes.c_int, ctypes.c_int, ctypes.c_int, P(ctypes.c_void_p)], ctypes.c_int),
            "me_comm_rank": ([ctypes.c_void_p, P(ctypes.c_int), P(ctypes.c_int)], ctypes.c_int),
            "me_comm_destroy": ([ctypes.c_void_p], None),
            "me_strerror": ([ctypes.c_int], ctypes.c_char_p),
            "me_last_error_detail": ([], ctypes.c_char_p),
            "me_version": ([], ctypes.c_char_p),
        }
        for name, (args, res) in sigs.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


# every symbol include/me.h declares (checked by tests/test_abi.py)
EXPORTS = ("me_estimate", "me_estimate_stage", "me_estimate_batch", "me_space_size", "me_decode", "me_plan_create", "me_plan_size", "me_plan_table_bytes",
           "me_plan_sweep", "me_plan_free", "me_sweep", "me_result_counts", "me_result_cap_counts",
           "me_result_columns", "me_result_copy_to_host", "me_result_status", "me_result_wait",
           "me_result_timing", "me_result_free", "me_result_rank", "me_result_digest", "me_digest_merge", "me_comm_check", "me_cyclic_block", "me_result_join", "me_partition", "me_join_counts", "me_comm_unique_id", "me_comm_init", "me_comm_rank",
           "me_comm_destroy", "me_strerror", "me_last_error_detail", "me_version")


def strerror(status: int) -> str:
    try:
        return lib().me_strerror(status).decode()
    except Exception:  # library not loadable: plain number
        return str(status)


def check(status: int, call: str):
    if status != ME_OK:
        detail = lib().me_last_error_detail().decode(errors="replace")
        raise MEError(status, call, detail)
