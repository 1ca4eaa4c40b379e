"""Benchmark of the estimator hot path (BASELINE.json metric: estimator
configs/sec at 1/2/4/8 B200, roofline fraction, bit-exact feasible set).

Workload: C5 = BASELINE.json configs[4], the synthetic Llama
grid (247,776 shapes) x world sizes 8..16384 x every 4D factorisation x
mbs 1..16 x seq 4K..128K x recompute x distributed optimizer, uneven PP
allowed, capacities 40/80/94/192 GiB -- 8.4e10 valid configurations, which the
north star partitions over the 8 GPUs of one box.  Every step sweeps ALL of
C5 whatever N is ("scaling": "strong"): the index space is cut into blocks of
CHUNK = 2^28 consecutive configs; at N = 1 each block is one me_plan_sweep
call; at N > 1 (default --partition cyclic) the blocks are dealt round-robin
by libme (me_cyclic_block: rank r sweeps blocks r, r + N, ... alone) and one
me_result_join per step joins them (NCCL allgather of every block's counts and
an exclusive scan on the device: global offsets).  --partition even: calls of
N * CHUNK configs, each split evenly over the ranks by the library with a join
per call.

A step = one pass of the whole hot path over the whole space: decode ->
estimate -> 80% filter -> order-preserving compaction into 64-byte records
(RECORDS; --mode full|index|count) -- every call's rows are written to HBM
(two caller buffers alternate).  The INDEX and COUNT modes are timed too and
reported under "modes".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--mode records|full|index|count]
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
    ap.add_argument("--no-modes", action="store_true", help="skip the INDEX / COUNT extra keys")
    ap.add_argument("--chunk-log2", type=int, default=28, help="configs per sweep call / cyclic block: 2^k")
    ap.add_argument("--no-verify", action="store_true", help="skip the untimed feasible-set digest check")
    ap.add_argument("--partition", default="cyclic", choices=["cyclic", "even"],
                    help="N>1: cyclic = libme's cyclic deal: rank r sweeps blocks r, r+N, ... of CHUNK configs "
                         "on its own and me_result_join joins every block's counts with one NCCL allgather per "
                         "step; even = every call covers N*CHUNK configs split evenly over the ranks by the "
                         "library (one join per call)")
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


def oracle_rate(sp, begin, end, threads, n, wins=4):
    """configs/s of the oracle (unchanged) over `wins` evenly spaced windows of
    n/wins configs of [begin, end).  The oracle walks its enumeration from
    index 0 to a window (table build + skip); that overhead is measured with a
    1-config window at the same offset and subtracted, so the rate counts the
    evaluation of the window's configurations only."""
    import oracle
    per = max(1, n // wins)
    done, net = 0, 0.0
    for w in range(wins):
        s = begin + (end - begin) * w // wins
        t = time.perf_counter()
        oracle.sweep(sp, s, s + 1, rows=False, threads=1)
        over = time.perf_counter() - t
        t = time.perf_counter()
        oracle.sweep(sp, s, s + per, rows=False, threads=threads)
        net += max(1e-9, time.perf_counter() - t - over)
        done += per
    return done / net, done, net


def cpu_baseline(sp, begin, end, budget_s=12.0):
    """The oracle (unchanged) on the host cores over a bounded, deterministic
    sample of the workload: evenly spaced windows of the bench range, with all
    host threads and with one thread."""
    import oracle
    threads = oracle.default_threads()
    r1, n1, t1 = oracle_rate(sp, begin, end, 1, 200_000)
    n = int(min(end - begin, max(1_000_000, r1 * threads * budget_s)))
    rate, done, el = oracle_rate(sp, begin, end, threads, n)
    return {"value": rate, "unit": "configs/s", "cores": threads, "kind": "oracle",
            "value_1thread": r1,
            "sample": f"4 evenly spaced windows of the first eighth of {WORKLOAD}: {done} configs on {threads} "
                      f"threads in {el:.1f} s and {n1} configs on 1 thread in {t1:.1f} s (survivor counts, every "
                      "estimator term evaluated; the oracle's table build and walk to each window are measured "
                      "with a 1-config window and subtracted)"}


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
        oracle.sweep(sp, s, s + 1, rows=False, threads=1)
        over = time.perf_counter() - t  # table build + walk to the window (subtracted)
        t = time.perf_counter()
        oracle.sweep(sp, s, s + per, rows=False, threads=threads)
        if i >= args.warmup:
            times.append(max(1e-9, time.perf_counter() - t - over))
    el = sum(times)
    v = per * args.steps / el
    line = {"impl": "reference", "metric": "estimator configs/sec", "value": v, "unit": "configs/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "config": {"workload": args.workload, "sample_per_step": per},
            "cpu_baseline": {"value": v, "unit": "configs/s", "cores": threads, "kind": "oracle",
                             "sample": f"{per} consecutive configs per step at evenly spaced offsets of the "
                                       f"first eighth of {args.workload} (the oracle's walk to each window, "
                                       "measured with a 1-config window, subtracted)"},
            "e2e": {"value": v, "unit": "configs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_steps(torch, dist, me, plan, calls, mode, ring, flush, stream, steps, warmup, world, comm, cyclic, n_blocks,
              clocks=None):
    """W untimed + K timed steps of the hot path; returns (ms max over ranks,
    per-call timings, this rank's survivors, the job's survivors) per step."""
    ncols = 0 if mode == me.ME_OUT_COUNT else 1

    def step():
        out = []
        for q, (b, e) in enumerate(calls):
            out.append(plan.sweep(b, e, mode=mode, out_cols=ring[q & 1] if ncols else None,
                                  comm=None if cyclic else comm,
                                  partition=me.ME_PART_CYCLIC if cyclic else me.ME_PART_EVEN))
        if cyclic:
            # a8: one NCCL allgather of every block's counts + device scan (libme)
            me.result_join(out, n_blocks, comm)
        return out

    def drain(results, timings=None):
        n_local = n_global = 0
        for i, r in enumerate(results):
            if r.status() != 0:
                raise RuntimeError("caller columns overflowed")
            lo, gl, off = r.counts()
            n_local += lo
            n_global = gl if cyclic else n_global + gl
            if timings is not None:
                timings.append(r.timing())
        for r in results:
            r.free()
        return n_local, n_global

    with torch.cuda.stream(stream):
        for _ in range(warmup):
            flush.zero_()
            drain(step())
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    timings = []
    import contextlib
    with (clocks if clocks is not None else contextlib.nullcontext()):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            ev0.record(stream)
            all_res = []
            for _ in range(steps):
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
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{torch.cuda.current_device()}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), timings, n_local // steps, n_global // steps


def verify_feasible_set(torch, dist, me, plan, calls, ring, stream, world, rank, workload):
    """Untimed: one more pass over this rank's calls in RECORDS mode, the
    order-dependent digest of each call's feasible set (me_result_digest),
    gathered and merged in index order (me_digest_merge) into the digest of
    the whole step's feasible set, compared with the oracle's per-chunk
    digests (tests/golden/<workload>_chunks.csv, written by
    tests/golden/gen_chunk_digests.py from oracle/)."""
    mine = []
    with torch.cuda.stream(stream):
        for q, (b, e) in enumerate(calls):
            r = plan.sweep(b, e, mode=me.ME_OUT_RECORDS, out_cols=ring[q & 1])
            if r.status() != 0:
                raise RuntimeError("caller columns overflowed")
            mine.append((b, r.counts()[0], r.cap_counts(), r.digest()))
            r.free()
    parts = [mine]
    if world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, mine)
    if rank != 0:
        return None
    allp = sorted(x for p_ in parts for x in p_)
    counts = [x[1] for x in allp]
    dig = me.digest_merge(counts, [x[3] for x in allp])
    out = {"survivors": sum(counts), "digest_index": f"{dig[0]:016x}", "digest_record": f"{dig[1]:016x}",
           "calls": len(allp)}
    gold = ROOT / "tests" / "golden" / f"{workload.lower()}_chunks.csv"
    if gold.exists():
        import csv
        with gold.open() as fh:
            g = {int(r["begin"]): r for r in csv.DictReader(fh)}
        if all(x[0] in g for x in allp) and len(g) == len(allp):
            rows = [g[x[0]] for x in allp]
            ref = me.digest_merge([int(r["count"]) for r in rows],
                                  [(int(r["digest_index"], 16), int(r["digest_record"], 16)) for r in rows])
            out["oracle_golden"] = str(gold.relative_to(ROOT))
            out["equal_to_oracle"] = (ref == dig and [int(r["count"]) for r in rows] == counts
                                      and all([int(r[f"cap{j}"]) for j in range(len(allp[0][2]))] == x[2]
                                              for r, x in zip(rows, allp)))
    return out


def ncu_summary():
    """per-kernel ncu figures of one C5 chunk at HEAD (scripts/ncu_summary.py)"""
    for name in ("r2_final", "r2b"):
        f = ROOT / "profiles" / name / "ncu_chunk40.json"
        if f.exists():
            return json.loads(f.read_text()), f"profiles/{name}/ncu_chunk40.json"
    return None, None


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    global CHUNK
    CHUNK = 1 << args.chunk_log2
    import torch
    import torch.distributed as dist

    import me_inputs as mi
    import paper_2411_06465_b200 as me

    rank, world, local = dist_env()
    assert world == args.gpus or world == 1, "launch N>1 with torchrun"
    torch.cuda.set_device(local)
    dev = local
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    modes = {"records": me.ME_OUT_RECORDS, "full": me.ME_OUT_FULL, "index": me.ME_OUT_INDEX, "count": me.ME_OUT_COUNT}
    mode = modes[args.mode]
    # u64 words written per survivor (FULL: 8 columns, RECORDS: one 64-byte row)
    words = {me.ME_OUT_RECORDS: 8, me.ME_OUT_FULL: 8, me.ME_OUT_INDEX: 1, me.ME_OUT_COUNT: 0}

    sp = mi.config(args.workload)
    stream = torch.cuda.Stream(device=dev)
    plan = me.Plan(sp, device=dev, stream=stream.cuda_stream)
    total = plan.size
    comm = me.Comm(dev) if world > 1 else None
    cyclic = world > 1 and args.partition == "cyclic"
    n_blocks = 0
    if cyclic:
        # a8 (libme): CHUNK-config blocks dealt round-robin (me_cyclic_block);
        # rank r sweeps blocks r, r + N, ... alone, one me_result_join per step
        calls, n_blocks = me.cyclic_blocks(0, total, CHUNK, rank, world)
    else:
        # N = 1: the space in CHUNK-config calls; N > 1 "even": calls of
        # N * CHUNK configs, each split evenly over the ranks by the library
        step_len = CHUNK * world
        calls = [(s, min(total, s + step_len)) for s in range(0, total, step_len)]

    def ring_for(m):
        return [out_buffers(torch, me, m, CHUNK + 64, device=dev) for _ in range(2)]

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    clocks = ClockSampler(dev)
    ring = ring_for(mode)
    ms_max, timings, surv_local, surv_global = run_steps(torch, dist, me, plan, calls, mode, ring, flush, stream,
                                                         args.steps, args.warmup, world, comm, cyclic, n_blocks,
                                                         clocks=clocks)
    del ring
    value = total * args.steps / (ms_max / 1e3)

    # per-kernel device times (CUDA events on the streams the kernels run on:
    # K0 rows + scan on the plan stream, the output kernel K3 on the sweep stream)
    rows_ms = sum(x[1] for x in timings)
    scan_ms = sum(x[2] for x in timings)
    out_ms = sum(x[3] for x in timings)
    n_launch = len(timings)
    peaks, peak_src = measured_peaks()
    ncu, ncu_src = ncu_summary()
    if mode != me.ME_OUT_COUNT:
        bytes_out = surv_local * 8 * words[mode] * args.steps
        achieved = bytes_out / (out_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": f"fused_kernel<{int(mode)},4> (K3: tests every configuration of the rows "
                                          "with survivors, writes every survivor row)",
                "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                "traffic": None, "peak_source": f"{peak_src} hbm_gbs (copy, MEASURED_PEAKS.json)",
                "algorithmic_bytes_per_launch": bytes_out / max(1, n_launch),
                "avg_launch_ms": out_ms / max(1, n_launch)}
        k3 = ncu and ncu["kernels"].get("fused_kernel")
        if k3:
            roof["traffic"] = k3["dram_bytes_read"] + k3["dram_bytes_write"]
            roof["traffic_note"] = (f"ncu DRAM bytes (read {k3['dram_bytes_read']:.4g} + write "
                                    f"{k3['dram_bytes_write']:.4g}) of K3 on C5 chunk {ncu['chunk']}, algorithmic "
                                    f"{ncu['algorithmic_write_bytes']} B for that launch ({ncu_src}); the reads are "
                                    "the 128-byte row entries of rows with survivors")
        mb = ROOT / "profiles" / "r1_v4" / "microbench.json"
        if mb.exists():
            w = json.loads(mb.read_text())["write_only_gbs"]
            roof["write_only_peak_gbs"] = w
            roof["frac_of_write_only"] = achieved / w
    else:
        roof = {"bound": "alu", "kernel": "rowcount_kernel (K0: every row, per-capacity survivor counts)",
                "achieved": None, "peak": None, "unit": "warp-instr/s", "frac": None, "traffic": 0}
    # integer-issue roofline (ncu, each kernel alone on the GPU: 148 SMs x 4
    # SMSPs x 1 warp-instruction / cycle)
    # integer-issue roofline per output mode (ncu --set full of C5 chunk 40,
    # each kernel alone on the GPU; 148 SMs x 4 SMSPs x 1 warp-instruction /
    # cycle): K0 and K3 of RECORDS, K3 of INDEX, K0 of COUNT
    issue = None
    if ncu:
        issue = {"chunk": ncu["chunk"], "configs": ncu["configs"],
                 "peak": "1 warp-instr / cycle / SMSP (148 x 4 x clock)"}
        for m_name in ("records", "index", "count"):
            f = ROOT / "profiles" / "r2_final" / f"ncu_chunk40_{m_name}.json"
            if not f.exists():
                continue
            d = json.loads(f.read_text())
            issue[m_name] = {"source": str(f.relative_to(ROOT))}
            for k in ("rowcount_kernel", "fused_kernel"):
                v = d["kernels"].get(k)
                if v:
                    issue[m_name][k] = {"issue_frac": v.get("issue_frac"), "warp_instr": v.get("warp_instr"),
                                        "warp_instr_per_config": v.get("warp_instr_per_config"),
                                        "pipe_alu_pct": v.get("pipe_alu_pct"), "pipe_fma_pct": v.get("pipe_fma_pct"),
                                        "duration_ms": v.get("duration_ms")}
        k0 = issue.get("count", {}).get("rowcount_kernel")
        if mode == me.ME_OUT_COUNT and k0:
            ach = k0["warp_instr"] / (k0["duration_ms"] / 1e3)
            roof.update({"achieved": ach, "unit": "warp-instr/s", "frac": k0["issue_frac"],
                         "peak": ach / k0["issue_frac"] if k0["issue_frac"] else None,
                         "peak_source": "148 SMs x 4 SMSPs x 1 warp-instruction per cycle at the capture's clock",
                         "traffic_note": "K0 alone (ncu, chunk 40, COUNT mode)"})
    line = {
        "metric": "estimator configs/sec", "value": value, "unit": "configs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": args.workload, "space_configs": total, "configs_per_gpu_per_step": total // world,
                   "per_step": "all of C5 (strong scaling)", "mode": args.mode, "chunk_configs": CHUNK,
                   "caps_gib": sp.caps_gb, "threshold": "4/5", "l2": "flushed (256 MiB write) before every step; "
                   "outputs (GBs per step) also exceed L2",
                   "parallelism": f"index-space partition x{world}" + (
                       f", libme cyclic blocks of {CHUNK} configs + me_result_join (NCCL allgather, device scan)"
                       if cyclic else (", libme even split per call" if world > 1 else ""))},
        "feasible_per_step": surv_global,
        "kernel_ms_per_step": {"rows_K0": rows_ms / args.steps, "scan": scan_ms / args.steps,
                               "output_K3": out_ms / args.steps},
        "roofline": roof,
        # per call: K0 rows, scan, K3 (COUNT: K0 alone); + the join kernel per step (N > 1)
        "gpu_launches": (3 if mode != me.ME_OUT_COUNT else 1) * n_launch + (args.steps if cyclic else 0),
        "clocks": clocks.summary(),
    }
    if issue:
        line["int_issue"] = issue
    # the other output modes on the same workload (extra keys)
    if not args.no_modes:
        extra = {}
        for name in ("index", "count"):
            if name == args.mode:
                continue
            m = modes[name]
            ring = ring_for(m)
            ms_m, tm, sl, sg = run_steps(torch, dist, me, plan, calls, m, ring, flush, stream, args.steps,
                                         args.warmup, world, comm, cyclic, n_blocks)
            del ring
            extra[name] = {"value": total * args.steps / (ms_m / 1e3), "unit": "configs/s",
                           "ms_per_step": ms_m / args.steps, "feasible_per_step": sg,
                           "kernel_ms_per_step": {"rows_K0": sum(x[1] for x in tm) / args.steps,
                                                  "scan": sum(x[2] for x in tm) / args.steps,
                                                  "output_K3": sum(x[3] for x in tm) / args.steps}}
        line["modes"] = extra

    # the step's feasible set against the oracle (untimed; bench calls of 2^28
    # configs = the golden chunks)
    if not args.no_verify and CHUNK == 1 << 28 and (world == 1 or cyclic):
        ring = ring_for(me.ME_OUT_RECORDS)
        fs = verify_feasible_set(torch, dist, me, plan, calls, ring, stream, world, rank, args.workload)
        del ring
        if fs is not None:
            line["feasible_set"] = fs

    # e2e: the public API with host buffers -- plan creation (host tables +
    # H2D) and a D2H of every survivor row inside the timed region
    if not args.no_e2e:
        e2e_ms, h2d, d2h = e2e_run(me, sp, dev, world, comm, calls, cyclic, n_blocks, mode, words[mode] > 0,
                                   args.e2e_steps, stream)
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        line["e2e"] = {"value": total * args.e2e_steps / (float(t.item()) / 1e3), "unit": "configs/s",
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps}
    if rank == 0 and not args.no_cpu:
        b0, e0 = unit_range(total, 0)
        line["cpu_baseline"] = cpu_baseline(sp, b0, e0)
    if comm:
        comm.check()
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


def e2e_run(me, sp, dev, world, comm, calls, cyclic, n_blocks, mode, rows_out, steps, stream):
    """End to end through the C ABI: host description in (plan creation: host
    tables + H2D), host rows out (D2H of every survivor row of this rank)."""
    import ctypes

    import torch
    HOST_ROWS = 1 << 26
    host = out_buffers(torch, me, mode, HOST_ROWS, pin_memory=True)
    ring = out_buffers(torch, me, mode, CHUNK + 64, device=dev)
    wd = 8 if mode in (me.ME_OUT_RECORDS, me.ME_OUT_FULL) else 1
    h2d = d2h = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        plan = me.Plan(sp, device=dev, stream=stream.cuda_stream)
        h2d += plan.table_bytes  # enumeration tables built on the host and uploaded
        results = []
        for (b, e) in calls:
            r = plan.sweep(b, e, mode=mode, out_cols=ring if rows_out else None, comm=None if cyclic else comm,
                           partition=me.ME_PART_CYCLIC if cyclic else me.ME_PART_EVEN)
            lo, gl, off = r.counts()
            if rows_out:
                arr = (ctypes.c_void_p * 8)(*([h.data_ptr() for h in host] + [None] * (8 - len(host))))
                for first in range(0, lo, HOST_ROWS):
                    n = min(HOST_ROWS, lo - first)
                    me.check(me.lib().me_result_copy_to_host(r.h, first, n, arr), "me_result_copy_to_host")
                d2h += lo * 8 * wd
            d2h += 8
            results.append(r)
        if cyclic:
            me.result_join(results, n_blocks, comm)
            results[0].counts()
            d2h += 8 * 17
        for r in results:
            r.free()
        plan.free()
    torch.cuda.synchronize()
    el = (time.perf_counter() - t0) * 1e3
    return el, h2d // steps, d2h // steps


if __name__ == "__main__":
    sys.exit(main())
