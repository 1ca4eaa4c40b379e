python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for c in 28 30 32; do timeout 600 python bench.py --mode count --steps 5 --warmup 3 --no-cpu --no-e2e --no-modes --no-verify --chunk-log2 $c 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d["value"]/1e9,1), round(d["ms_per_step"],2), {k: round(v,1) for k,v in d["kernel_ms_per_step"].items()})'; done
python - <<'PY'
import time, torch, me_inputs as mi, paper_2411_06465_b200 as me
sp = mi.config("C5"); s = torch.cuda.Stream(); plan = me.Plan(sp, device=0, stream=s.cuda_stream)
with torch.cuda.stream(s):
    for rep in range(3):
        t = time.perf_counter(); rs = [plan.sweep(k << 28, (k + 1) << 28, mode=me.ME_OUT_COUNT) for k in range(100)]; t1 = time.perf_counter()
        torch.cuda.synchronize(); t2 = time.perf_counter()
        for r in rs: r.free()
        print("host enqueue per call us", (t1 - t) / 100 * 1e6, "gpu drain", (t2 - t1) * 1e3, "ms")
PY
