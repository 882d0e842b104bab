"""Summarise ncu evidence for profiles/ (run here, on the CPU box).

    python scripts/ncu_summary.py full  gpurun_out/prof_k_score.ncu-rep  ROWS_PER_LAUNCH  > profiles/x.md
    python scripts/ncu_summary.py launches gpurun_out/launches.csv                         > profiles/y.md

`full`: key metrics of a `ncu --set full` capture (duration, DRAM bytes and
throughput, pipe utilisation, issue, occupancy, stall mix) per launch, and the
DRAM traffic per scored row (written to profiles/k_score_traffic.json when
--traffic is given). `launches`: per-kernel share of device time from a
`--metrics gpu__time_duration.sum` launch list.
"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes_read.sum.per_second", "DRAM read BW"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
]


def _raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    return rows[0], rows[1], rows[2:]


def full(rep: str, rows_per_launch: int, traffic_out: str | None) -> None:
    hdr, units, data = _raw(rep)
    col = {h: i for i, h in enumerate(hdr)}
    names = [d[col["Kernel Name"]].split("(")[0] for d in data]
    print(f"### ncu --set full: `{rep.split('/')[-1]}`\n")
    print(f"kernel: `{names[0]}` ({len(data)} launches profiled, {rows_per_launch} rows per launch)\n")
    print("| metric | unit | " + " | ".join(f"launch {i}" for i in range(len(data))) + " |")
    print("|---|---|" + "---|" * len(data))
    for k, label in KEYS:
        if k in col:
            print(f"| {label} (`{k}`) | {units[col[k]]} | " + " | ".join(d[col[k]] for d in data) + " |")
    d = data[0]
    st = [(h.split("stalled_")[1], float(d[i])) for h, i in col.items()
          if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued") and d[i]]
    tot = sum(v for _, v in st) or 1.0
    print("\nstall sampling (launch 0): " + ", ".join(f"{n} {100 * v / tot:.1f}%" for n, v in
                                                   sorted(st, key=lambda x: -x[1])[:8]))
    rd = float(d[col["dram__bytes_read.sum"]]) * (1e9 if units[col["dram__bytes_read.sum"]] == "Gbyte" else 1e6)
    wr = float(d[col["dram__bytes_write.sum"]]) * (1e6 if units[col["dram__bytes_write.sum"]] == "Mbyte" else 1e3)
    dur_s = float(d[col["gpu__time_duration.sum"]]) * (1e-6 if units[col["gpu__time_duration.sum"]] == "us" else 1e-3)
    per_row = (rd + wr) / rows_per_launch
    print(f"\nDRAM traffic per launch: {(rd + wr) / 1e9:.4f} GB = {per_row:.1f} B/row "
          f"(algorithmic 2V+26 = {2 * 151936 + 26} B/row at V=151936); {rd / dur_s / 1e9:.0f} GB/s read under ncu "
          f"(cold, serialised, clock as listed).")
    if traffic_out:
        # stamped with the digest of the kernel's sources: bench.py quotes the
        # capture only while the sources are the ones it was taken on
        sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
        # the SASS digest of the binary the capture was taken on (written next to
        # the report on the GPU box by scripts/gpu_round2b.sh), else of the local build
        import pathlib
        stamp_file = pathlib.Path(rep).with_name("k_score_sass_stamp.txt")
        if stamp_file.exists():
            stamp = stamp_file.read_text().strip()
        else:
            from bench import k_score_stamp
            stamp = k_score_stamp()
        json.dump({"source": rep.split("/")[-1], "kernel": names[0], "rows_per_launch": rows_per_launch,
                   "dram_bytes_per_launch": rd + wr, "dram_bytes_per_row": per_row,
                   "sass_stamp": stamp}, open(traffic_out, "w"), indent=1)


def launches(path: str) -> None:
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[i], rows[i + 1:]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").strip()
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    step = {n: v for n, v in tot.items() if "gen_logits" not in n}
    T, Ts = sum(tot.values()), sum(step.values())
    print(f"### launch list `{path.split('/')[-1]}` (gpu__time_duration.sum, cold/serialised)\n")
    print("| kernel | launches | total ns | share of all | share of step (excl. synthetic LM head) |")
    print("|---|---|---|---|---|")
    for n, v in sorted(tot.items(), key=lambda x: -x[1]):
        s = f"{100 * v / Ts:.2f}%" if n in step else "— (warm-up generator, not timed)"
        print(f"| `{n[:70]}` | {cnt[n]} | {v:.0f} | {100 * v / T:.2f}% | {s} |")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], int(sys.argv[3]), sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        launches(sys.argv[2])
