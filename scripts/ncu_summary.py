"""Summarise an ncu --set full capture of one C5 chunk (scripts/gpu_prof.sh)
into the per-kernel JSON bench.py reads (profiles/ncu_chunk40.json):
  python scripts/ncu_summary.py gpurun_out/prof.ncu-rep gpurun_out/chunk40.json > profiles/ncu_chunk40.json"""
import csv
import io
import json
import subprocess
import sys

rep, chunk_json = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
SCALE = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "byte": 1.0, "Kbyte": 1e3,
         "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}  # durations -> ms, sizes -> bytes
chunk = json.loads(open(chunk_json).read().strip().splitlines()[-1])
configs = chunk["end"] - chunk["begin"]
rounds = configs / 32


def f(d, k):
    try:
        return float(d[k].replace(",", "")) * SCALE.get(units[hdr.index(k)], 1.0)
    except (KeyError, ValueError):
        return None


out = {"chunk": chunk["chunk"], "mode": chunk.get("mode"), "configs": configs, "survivors": chunk["survivors"],
       "algorithmic_write_bytes": chunk["algorithmic_write_bytes"], "kernels": {},
       "note": "one ncu --set full capture (serialised, cold caches, --clock-control none) of the kernels of "
               "C5 chunk 40 (scripts/profile_chunk.py 40); DRAM bytes vs the algorithmic bytes of the same launch"}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("me::", "").replace("<unnamed>::", "")
    name = name.replace("unnamed>::", "").replace("(anonymous namespace)::", "")
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): f(d, k) for k in hdr
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(v for v in stalls.values() if v) or 1
    inst = f(d, "smsp__inst_executed.sum")
    tinst = f(d, "smsp__thread_inst_executed.sum") or f(d, "sm__sass_thread_inst_executed.sum")
    cyc = f(d, "sm__cycles_elapsed.avg")
    nsm = f(d, "device__attribute_multiprocessor_count") or 148
    base = name.split("<")[0]
    if base in out["kernels"] and (out["kernels"][base].get("duration_ms") or 0) >= (f(d, "gpu__time_duration.sum") or 0):
        continue  # keep the longest launch of each kernel
    name = base
    out["kernels"][name] = {
        "warp_instr": inst, "warp_instr_per_config": inst / configs if inst else None,
        "thread_instr_per_config": tinst / configs if tinst else None,
        "pipe_alu_pct": f(d, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "pipe_fma_pct": f(d, "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
        "issue_frac": inst / (cyc * nsm * 4) if inst and cyc else None,
        "duration_ms": f(d, "gpu__time_duration.sum"),
        "dram_bytes_read": f(d, "dram__bytes_read.sum"), "dram_bytes_write": f(d, "dram__bytes_write.sum"),
        "issue_active_pct": f(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": f(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "inst_executed": inst, "warp_instr_per_round": inst / rounds if inst else None,
        "regs": f(d, "launch__registers_per_thread"),
        "top_stalls": {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -(x[1] or 0))[:5]},
    }
print(json.dumps(out, indent=1))
