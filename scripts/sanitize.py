"""Small sweeps through every kernel path, for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck; scripts/gpu_sanitize.sh).  Checks each result
against the oracle so a run that stays silent under the tools is also right."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import me_inputs as mi  # noqa: E402
import oracle  # noqa: E402
import paper_2411_06465_b200 as me  # noqa: E402

torch.cuda.set_device(0)
spaces = [
    ("C1", mi.config("C1")),
    ("gbs", mi.Space(models=mi.random_models(3, seed=21, small=True), world=[6, 8, 12], caps_gb=[1, 2, 4],
                     mbs=[1, 2, 3], seq=[8, 12, 16, 24], gbs=96, uneven=1, thr_num=9, thr_den=10)),
    ("stage_max", mi.Space(models=mi.random_models(4, seed=23), world=[8, 24], caps_gb=[24, 40, 80, 192],
                           mbs=[1, 2], seq=[4096, 32768], uneven=1, stage_max=1)),
    ("vpp_sp_off", mi.Space(models=mi.random_models(4, seed=53), world=[16, 24], caps_gb=[24, 80], mbs=[1, 2],
                            seq=[4096], vpp=2, gbs=768, sp_off=1)),
    ("masks8", mi.Space(models=mi.random_models(3, seed=22), world=[12, 48], caps_gb=[24, 40, 80, 94, 141, 180, 192, 288],
                        mbs=[1, 8], seq=[2048, 32768], rc_mask=2, do_mask=1)),
]
bad = 0
for name, sp in spaces:
    idx, rows, n, caps = oracle.sweep(sp, threads=4)
    plan = me.Plan(sp)
    for mode in (me.ME_OUT_COUNT, me.ME_OUT_INDEX, me.ME_OUT_FULL, me.ME_OUT_RECORDS):
        for (b, e) in ((0, 0), (3, plan.size - 2)):
            r = plan.sweep(b, e, mode=mode)
            e2 = e or plan.size
            ri, rr, rn, rc = oracle.sweep(sp, b, e2, threads=4)
            ok = r.counts()[0] == rn and r.cap_counts() == rc
            if mode:
                got = r.to_host()
                ok &= bool(np.array_equal(got["index_mask"], ri))
                if mode >= 2:
                    ok &= bool(np.array_equal(got["total"], rr[:, 6]))
                    ok &= r.digest() == oracle.digest_of_rows(ri, rr)
                    if mode == me.ME_OUT_RECORDS and len(sp.cap_bytes) >= 2:
                        r.rank(green_cap=0, yellow_cap=1, gpus_per_node=8, k=3)
            bad += not ok
            print(name, mode, (b, e), "ok" if ok else "MISMATCH", flush=True)
            r.free()
    plan.free()
rows_, mask_, st_ = me.me_estimate_batch([mi.PRESETS["llama3.1-8b"]], None,
                                         [dict(d=2, t=2, p=2, c=2, b=1, s=8192, gbs=64)], caps_bytes=[40 << 30])
me.me_estimate_stage(mi.PRESETS["llama3.1-8b"], me.STAGE_ARGMAX, d=2, t=2, p=4, c=1, b=1, s=8192)
print("SANITIZE", "OK" if not bad else f"{bad} MISMATCHES", os.environ.get("ME_MAX_ROWS", ""))
sys.exit(1 if bad else 0)
