"""Transcribe the paper's ten result tables into tests/golden/paper_tables.csv.

Run ONCE, here, against the read-only paper text (PAPER.md of arXiv 2411.06465);
the CSV it writes is committed and is the only thing the tests read (the paper
text does not exist on the GPU box).  Every row is a printed cell: nothing here
is computed from the oracle or from the CUDA path.

Tables (PAPER.md line of the caption):
  est_a100_8b_s8192   P:420  "Estimated Total Memory ... Llama-3.1-8B on A100(40GB) ... 8,192"
  thr_a100_8b_s8192   P:458  "Measured throughput ... Llama-3.1-8B on A100 (40GB) ... 8,192"
  thr_h100_8b_s8192   P:515  "Measured throughput ... Llama-3.1-8B on H100 (94GB) ... 8,192"
  est_a100_70b_s8192  P:628  "Estimated ... Llama-3.1-70B on A100(40GB) ... 8,192"
  thr_a100_70b_s8192  P:653  "Measured ... Llama-3.1-70B on A100 (40GB) ... 8,192"
  est_h100_8b_s8192
  est_h100_8b_s16384
  est_h100_8b_s32768
  thr_h100_8b_s16384
  thr_h100_8b_s32768

CSV columns: table, kind (est|thr), model (llama3.1-8b|llama3.1-70b), gpu_gb,
seq, tp, cp, pp, mbs, n_gpus, text (the printed cell text), colour
(green|yellow|red), line (PAPER.md line of the row).
"""
import csv
import re
import sys
from pathlib import Path

PAPER = Path(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/PAPER.md")
OUT = Path(__file__).with_name("paper_tables.csv")

ROW = re.compile(r"^\s*\((\d+),\s*(\d+),\s*(\d+),\s*(\d+)\)\s*&(.*)$")
CELL = re.compile(r"\\cellcolor\{light(green|yellow|red)\}\s*(?:\\textbf\{)?\s*([0-9.]+|OOM)\}?")


def main():
    lines = PAPER.read_text().splitlines()
    rows = []
    i = 0
    while i < len(lines):
        ln = lines[i]
        m = re.search(r"\\caption\{(Estimated Total Memory|Measured throughput)", ln)
        if not m:
            i += 1
            continue
        kind = "est" if m.group(1).startswith("Estimated") else "thr"
        model = "llama3.1-70b" if "70B" in ln else "llama3.1-8b"
        gpu_gb = 94 if "H100" in ln else 40
        seq = int(re.search(r"(8,192|16,384|32,768)", ln).group(1).replace(",", ""))
        gpu = "h100" if gpu_gb == 94 else "a100"
        name = f"{kind}_{gpu}_{model.split('-')[1]}_s{seq}"
        # header row with GPU counts
        j = i + 1
        while "GPUs" not in lines[j]:
            j += 1
        counts = [int(x) for x in re.findall(r"(\d+) GPUs", lines[j])]
        j += 1
        while "\\end{tabular}" not in lines[j]:
            r = ROW.match(lines[j])
            if r:
                tp, cp, pp, mbs = (int(r.group(k)) for k in range(1, 5))
                cells = [c.strip() for c in r.group(5).replace("\\\\", "").replace("\\hline", "").split("&")]
                assert len(cells) == len(counts), (j + 1, cells, counts)
                for n, c in zip(counts, cells):
                    if c.strip() in ("-", ""):
                        continue
                    cm = CELL.search(c)
                    assert cm, (j + 1, c)
                    rows.append(dict(table=name, kind=kind, model=model, gpu_gb=gpu_gb, seq=seq,
                                     tp=tp, cp=cp, pp=pp, mbs=mbs, n_gpus=n, text=cm.group(2),
                                     colour=cm.group(1), line=j + 1))
            j += 1
        i = j
    with OUT.open("w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=list(rows[0].keys()))
        w.writeheader()
        w.writerows(rows)
    by = {}
    for r in rows:
        by[r["table"]] = by.get(r["table"], 0) + 1
    print(by, len(rows))


if __name__ == "__main__":
    main()
