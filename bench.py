"""Benchmark of the estimator hot path (BASELINE.json metric: estimator
configs/sec at 1/2/4/8 B200, roofline fraction, bit-exact feasible set).

Workload: C5 = BASELINE.json configs[4], the synthetic Llama
grid (247,776 shapes) x world sizes 8..16384 x every 4D factorisation x
mbs 1..16 x seq 4K..128K x recompute x distributed optimizer, uneven PP
allowed, capacities 40/80/94/192 GiB -- 8.4e10 valid configurations, which the
north star partitions over the 8 GPUs of one box.  Every step sweeps ALL of
C5 whatever N is ("scaling": "strong"): the index space is cut into calls of
N * CHUNK consecutive configs and each call is split evenly over the ranks.

A step = one pass of the whole hot path over the whole space: decode ->
estimate -> 80% filter -> order-preserving compaction into FULL records
(8 u64 columns) -- every call's columns are written to HBM (two column sets
alternate) -- with the NCCL allgather of the per-call survivor counts (global
offsets) when N > 1.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--mode full|index|count]
  python bench.py --impl reference ...   (the CPU oracle on the host cores)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CHUNK = 1 << 28          # configs per rank per me_plan_sweep call
UNITS = 8                # C5 split into 8 equal units (used for the CPU baseline sample)
WORKLOAD = "C5"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--mode", default="records", choices=["records", "full", "index", "count"])
    ap.add_argument("--workload", default=WORKLOAD)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--partition", default="cyclic", choices=["cyclic", "even"],
                    help="N>1: cyclic = rank r sweeps calls r, r+N, ... of CHUNK configs on its own and the "
                         "per-call counts are joined by one allgather per step; even = every call covers "
                         "N*CHUNK configs split evenly over the ranks by the library (one join per call)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def unit_range(total, unit):
    return total * unit // UNITS, total * (unit + 1) // UNITS


class ClockSampler:
    """NVML clocks and throttle reasons sampled during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device):
        self.samples, self.reasons = [], set()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def cpu_baseline(sp, begin, end, budget_s=12.0):
    """The oracle (unchanged) on the host cores over a bounded, deterministic
    sample of the workload: evenly spaced windows of the bench range."""
    import oracle
    threads = oracle.default_threads()
    # calibrate
    t = time.perf_counter()
    cal = 1_000_000
    oracle.sweep(sp, begin, begin + cal, rows=False, threads=threads)
    dt = time.perf_counter() - t
    rate = cal / max(dt, 1e-6)
    n = int(min(end - begin, max(cal, rate * budget_s)))
    wins = 4
    per = max(1, n // wins)
    done, t0 = 0, time.perf_counter()
    for w in range(wins):
        s = begin + (end - begin) * w // wins
        oracle.sweep(sp, s, s + per, rows=False, threads=threads)
        done += per
    el = time.perf_counter() - t0
    return {"value": done / el, "unit": "configs/s", "cores": threads, "kind": "oracle",
            "sample": f"{wins} evenly spaced windows of {per} configs of the first eighth of {WORKLOAD} "
                      f"(survivor counts, all estimator terms evaluated), {done} configs in {el:.1f} s"}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    import me_inputs as mi
    import oracle
    sp = mi.config(args.workload)
    total = oracle.space_size(sp)
    b, e = unit_range(total, 0)
    threads = oracle.default_threads()
    per = 2_000_000
    times = []
    for i in range(args.warmup + args.steps):
        s = b + (e - b) * (i % 97) // 97
        t = time.perf_counter()
        oracle.sweep(sp, s, s + per, rows=False, threads=threads)
        if i >= args.warmup:
            times.append(time.perf_counter() - t)
    el = sum(times)
    v = per * args.steps / el
    line = {"impl": "reference", "metric": "estimator configs/sec", "value": v, "unit": "configs/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "config": {"workload": args.workload, "sample_per_step": per},
            "cpu_baseline": {"value": v, "unit": "configs/s", "cores": threads, "kind": "oracle",
                             "sample": f"{per} consecutive configs per step at evenly spaced offsets of the "
                                       f"first eighth of {args.workload}"},
            "e2e": {"value": v, "unit": "configs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import me_inputs as mi
    import paper_2411_06465_b200 as me
    from paper_2411_06465_b200.cyclic import cyclic_calls, cyclic_join, n_calls

    rank, world, local = dist_env()
    assert world == args.gpus or world == 1, "launch N>1 with torchrun"
    torch.cuda.set_device(local)
    dev = local
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    mode = {"records": me.ME_OUT_RECORDS, "full": me.ME_OUT_FULL, "index": me.ME_OUT_INDEX,
            "count": me.ME_OUT_COUNT}[args.mode]
    # u64 words written per survivor (FULL: 8 columns, RECORDS: one 64-byte row)
    ncols = {me.ME_OUT_RECORDS: 8, me.ME_OUT_FULL: 8, me.ME_OUT_INDEX: 1, me.ME_OUT_COUNT: 0}[mode]

    sp = mi.config(args.workload)
    stream = torch.cuda.Stream(device=dev)
    plan = me.Plan(sp, device=dev, stream=stream.cuda_stream)
    total = plan.size
    # this job: units 0..world-1; each me_plan_sweep call covers world*CHUNK
    # consecutive configs, split evenly over the ranks by the library
    job_b, job_e = 0, total
    calls = []
    s = job_b
    while s < job_e:
        e = min(job_e, s + CHUNK * world)
        calls.append((s, e))
        s = e
    comm = me.Comm(dev) if world > 1 else None
    calls_even = calls
    cyclic = world > 1 and args.partition == "cyclic"
    if cyclic:
        # whole CHUNK-config calls dealt round-robin: neighbouring chunks have
        # similar survivor density, so every rank writes about as many rows,
        # and no rank waits for the others until the step's single join
        calls = cyclic_calls(job_b, job_e, CHUNK, rank, world)
        calls_total = n_calls(job_b, job_e, CHUNK)
    sweep_comm = None if cyclic else comm

    def join(results):
        """a8 for the cyclic partition: one allgather of every call's count"""
        return cyclic_join([r.counts()[0] for r in results], calls_total, world, device=dev)

    ring = [out_buffers(torch, me, mode, CHUNK + 64, device=dev) for _ in range(2)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step(collect=None):
        out = []
        for q, (b, e) in enumerate(calls):
            r = plan.sweep(b, e, mode=mode, out_cols=ring[q & 1] if ncols else None, comm=sweep_comm)
            out.append(r)
        if cyclic:
            joined.append(join(out)[2])
        return out

    joined = []

    def drain(results, timings=None):
        n_local = n_global = 0
        for r in results:
            if r.status() != 0:
                raise RuntimeError("caller columns overflowed")
            lo, gl, off = r.counts()
            n_local += lo
            n_global += gl
            if timings is not None:
                timings.append(r.timing())
            r.free()
        return n_local, n_global

    # warmup
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            flush.zero_()
            drain(step())
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev)
    timings = []
    with clocks:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            ev0.record(stream)
            all_res = []
            for _ in range(args.steps):
                flush.zero_()
                all_res.append(step())
            ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    n_local = n_global = 0
    for res in all_res:
        lo, gl = drain(res, timings)
        n_local += lo
        n_global += gl
    if cyclic:
        n_global = sum(joined[-args.steps:])
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    configs = (job_e - job_b) * args.steps
    value = configs / (ms_max / 1e3)

    # per-kernel device times (CUDA events on the sweep stream)
    count_ms = sum(x[1] for x in timings)
    write_ms = sum(x[3] for x in timings)
    scan_ms = sum(x[2] for x in timings)
    n_launch = len(timings)
    survivors_local_per_step = n_local // args.steps
    peaks, peak_src = measured_peaks()
    # per-kernel ncu summary of one C5 chunk (scripts/gpu_prof.sh +
    # scripts/ncu_summary.py): DRAM traffic and warp instructions per round
    ncu = ROOT / "profiles" / "ncu_chunk40.json"
    ncu_k = json.loads(ncu.read_text()).get("kernels", {}) if ncu.exists() else {}
    ncu_c = json.loads(ncu.read_text()) if ncu.exists() else {}

    def ncu_kernel(prefix):
        return next((v for k, v in ncu_k.items() if k.startswith(prefix)), None)

    # integer-issue roofline of the pass that evaluates every config (the
    # stage kernel K1; COUNT mode: the count kernel): warp instructions per
    # round of 32 configs from the ncu capture x this rank's rounds, over the
    # pass's CUDA-event time (with overlapped passes that time includes
    # sharing the SMs with the previous sub-range's expand kernel)
    issue = None
    kname = "count_kernel" if mode == me.ME_OUT_COUNT else "stage_kernel"
    kk = ncu_kernel(kname)
    ipr = kk and kk.get("warp_instr_per_round")
    if ipr and count_ms > 0:
        clock = peaks.get("sm_max_mhz", 1965.0) * 1e6
        issue_peak = 148 * 4 * clock
        ach = (job_e - job_b) // world * args.steps / 32 * ipr / (count_ms / 1e3)
        issue = {"bound": "alu", "kernel": f"{kname} (evaluates every config)", "achieved": ach,
                 "peak": issue_peak, "unit": "warp-instr/s", "frac": ach / issue_peak, "traffic": 0,
                 "instr_per_round_ncu": ipr,
                 "peak_source": "148 SMs x 4 SMSPs x 1 warp-instr/cycle x sm_max_mhz (MEASURED_PEAKS.json)"}
    if mode != me.ME_OUT_COUNT:
        bytes_write = survivors_local_per_step * 8 * ncols * args.steps
        achieved = bytes_write / (write_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": f"expand_kernel<{int(mode)},4> (writes every survivor row)",
                "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                "traffic": None, "peak_source": f"{peak_src} hbm_gbs (copy)",
                "algorithmic_bytes_per_launch": bytes_write / max(1, n_launch),
                "avg_launch_ms": write_ms / max(1, n_launch)}
        ek = ncu_kernel("expand_kernel")
        if ek:
            roof["traffic"] = ek["dram_bytes_read"] + ek["dram_bytes_write"]
            roof["traffic_note"] = (f"ncu DRAM bytes (read {ek['dram_bytes_read']:.4g} + write "
                                    f"{ek['dram_bytes_write']:.4g}) of the expand kernel of C5 chunk "
                                    f"{ncu_c['chunk']}, algorithmic {ncu_c['algorithmic_write_bytes']} B for that "
                                    "launch; the reads are the 8-byte survivor descriptors and the row table")
        mb = ROOT / "profiles" / "r1_v4" / "microbench.json"
        if mb.exists():
            w = json.loads(mb.read_text())["write_only_gbs"]
            roof["write_only_peak_gbs"] = w
            roof["frac_of_write_only"] = achieved / w
        if issue:
            roof["stage_pass_issue"] = issue
    else:
        roof = issue or {"bound": "alu", "kernel": "count_kernel<4> (count pass)", "achieved": None, "peak": None,
                         "unit": "warp-instr/s", "frac": None, "traffic": 0}
    line = {
        "metric": "estimator configs/sec", "value": value, "unit": "configs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": args.workload, "space_configs": total, "configs_per_gpu_per_step": (job_e - job_b) // world,
                   "per_step": "all of C5 (strong scaling)", "mode": args.mode, "chunk_configs_per_rank": CHUNK,
                   "caps_gib": sp.caps_gb, "threshold": "4/5", "l2": "flushed (256 MiB write) before every step; "
                   "outputs (GBs per step) also exceed L2", "parallelism": f"index-space partition x{world}"
                   + (f", {args.partition} calls of {CHUNK} configs" if world > 1 else "")},
        "feasible_per_step": n_global // args.steps,
        "kernel_ms_per_step": {"count": count_ms / args.steps, "scan": scan_ms / args.steps,
                               "write": write_ms / args.steps},
        "roofline": roof,
        # per sub-range: row, stage, scan, expand kernels (COUNT: count, scan)
        "gpu_launches": 4 * n_launch if mode != me.ME_OUT_COUNT else 2 * n_launch,
        "clocks": clocks.summary(),
    }

    # e2e: the public API with host buffers -- plan creation (host tables +
    # H2D) and a D2H of every survivor column inside the timed region
    if not args.no_e2e:
        e2e_ms, h2d, d2h = e2e_run(me, sp, dev, world, comm, calls_even, mode, ncols, args.e2e_steps, stream)
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        line["e2e"] = {"value": (job_e - job_b) * args.e2e_steps / (float(t.item()) / 1e3), "unit": "configs/s",
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps}
    if rank == 0 and not args.no_cpu:
        b0, e0 = unit_range(total, 0)
        line["cpu_baseline"] = cpu_baseline(sp, b0, e0)
    if comm:
        comm.destroy()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def out_buffers(torch, me, mode, rows, **kw):
    """Output buffers of `rows` survivors: 8 columns (FULL; one allocation cut
    into adjacent slices), 1 column (INDEX), one array of 64-byte records
    (RECORDS) or none (COUNT)."""
    if mode == me.ME_OUT_COUNT:
        return []
    if mode == me.ME_OUT_INDEX:
        return [torch.empty(rows, dtype=torch.int64, **kw)]
    flat = torch.empty(8 * rows, dtype=torch.int64, **kw)
    return [flat] if mode == me.ME_OUT_RECORDS else list(flat.view(8, rows).unbind(0))


def e2e_run(me, sp, dev, world, comm, calls, mode, ncols, steps, stream):
    """End to end through the C ABI: host description in, host columns out."""
    import ctypes

    import torch
    HOST_ROWS = 1 << 26
    host = out_buffers(torch, me, mode, HOST_ROWS, pin_memory=True)
    ring = out_buffers(torch, me, mode, CHUNK + 64, device=dev)
    h2d = d2h = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        plan = me.Plan(sp, device=dev, stream=stream.cuda_stream)
        h2d += plan.table_bytes  # enumeration tables built on the host and uploaded
        for (b, e) in calls:
            r = plan.sweep(b, e, mode=mode, out_cols=ring if ncols else None, comm=comm)
            lo, gl, off = r.counts()
            if ncols:
                arr = (ctypes.c_void_p * 8)(*([h.data_ptr() for h in host] + [None] * (8 - len(host))))
                for first in range(0, lo, HOST_ROWS):
                    n = min(HOST_ROWS, lo - first)
                    me.check(me.lib().me_result_copy_to_host(r.h, first, n, arr), "me_result_copy_to_host")
                d2h += lo * 8 * ncols
            d2h += 8
            r.free()
        plan.free()
    torch.cuda.synchronize()
    el = (time.perf_counter() - t0) * 1e3
    return el, h2d // steps, d2h // steps


if __name__ == "__main__":
    sys.exit(main())
