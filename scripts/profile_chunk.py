"""One RECORDS (or FULL: second argument "full") sweep call of bench.py's launch configuration (C5, one 2^28-config
chunk), for ncu: prints the chunk's survivors so the profiled write kernel's
DRAM traffic can be set against its algorithmic bytes (survivors x 64 B)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import me_inputs as mi  # noqa: E402
import paper_2411_06465_b200 as me  # noqa: E402

CHUNK = 1 << 28
k = int(sys.argv[1]) if len(sys.argv) > 1 else 40
mode = {"full": me.ME_OUT_FULL, "index": me.ME_OUT_INDEX, "count": me.ME_OUT_COUNT}.get(
    sys.argv[2] if len(sys.argv) > 2 else "records", me.ME_OUT_RECORDS)
sp = mi.config("C5")
stream = torch.cuda.Stream()
plan = me.Plan(sp, device=0, stream=stream.cuda_stream)
if mode == me.ME_OUT_FULL:
    cols = [torch.empty(CHUNK + 64, dtype=torch.int64, device="cuda") for _ in range(8)]
elif mode == me.ME_OUT_INDEX:
    cols = [torch.empty(CHUNK + 64, dtype=torch.int64, device="cuda")]
elif mode == me.ME_OUT_COUNT:
    cols = None
else:
    cols = [torch.empty(8 * (CHUNK + 64), dtype=torch.int64, device="cuda")]
with torch.cuda.stream(stream):
    r = plan.sweep(k * CHUNK, (k + 1) * CHUNK, mode=mode, out_cols=cols)
    n = r.counts()[0]
    ms = r.timing()
print(json.dumps({"chunk": k, "mode": int(mode), "begin": k * CHUNK, "end": (k + 1) * CHUNK, "configs": CHUNK,
                  "survivors": n,
                  "algorithmic_write_bytes": n * {me.ME_OUT_INDEX: 8, me.ME_OUT_COUNT: 0}.get(mode, 64), "timing_ms": ms}))
