"""Single-GPU projection of the 1/2/4/8-GPU scaling curve.

The path has no data-path collective: each rank scores its own LPT shard of
whole groups and the ranks meet once per step in a 2.6 KB all-reduce of the
partials. So the N-GPU step time is the slowest rank's shard time plus that
all-reduce. This script times every rank's shard of the N-rank layout one
after another on the one B200 (the same `prorl_score_host` call, resident
logits pool, CUDA events on the stream) and reports, per N:

  * strong scaling (the C4 batch, BASELINE's "8-GPU group-sharded" config,
    split over N ranks): projected masked tok/s = all rows / max rank time;
  * weak scaling (a C3-sized shard per rank, the bench's default):
    projected masked tok/s = all rows / max rank time;
  * the LPT imbalance (max / mean active rows) and max / mean rank time.

It is a projection, not a measurement of N GPUs: it assumes every GPU runs at
this one's clock and adds nothing for the all-reduce (~20 us per step over
NVLink against 100+ ms steps). Run on the GPU box:

    python scripts/scaling_projection.py > profiles/r02_scaling_projection.md
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2603_18815_b200 import synth  # noqa: E402
from paper_2603_18815_b200.hotpath import ScoreConfig, Scorer  # noqa: E402

MB = 16576
STEPS = 3


def rank_time(sc: Scorer, shard, c: dict, pool) -> float:
    cfg = ScoreConfig(vocab=c["vocab"], dtype=c["dtype"], microbatch_rows=MB)
    host = shard.batch.pinned()
    sc.score_host(host, cfg, pool, fill=True, seed=2603)  # fills the pool (LM-head stand-in)
    sc.score_host(host, cfg, pool, fill=False, seed=2603)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(STEPS):
        sc.score_host(host, cfg, pool, fill=False, seed=2603)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / STEPS / 1e3


def main() -> None:
    sc = Scorer(0)
    pool = [torch.empty((MB, 151936), dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    print("### Scaling projection from per-rank shard times on one B200 (`scripts/scaling_projection.py`)\n")
    print("Each rank's LPT shard of the N-rank layout timed on the same GPU (resident logits pool, "
          f"{STEPS} steps each); projected N-GPU throughput = all active rows / the slowest rank's step time "
          "(no data-path collective; the 2.6 KB partials all-reduce is not added). A projection, not an N-GPU "
          "measurement.\n")
    for scaling, cname in (("strong", "c4"), ("weak", "c3")):
        base = synth.CONFIGS[cname]
        print(f"#### {scaling} scaling, {cname} ({base['desc']})\n")
        print("| N | active rows (all ranks) | LPT imbalance (rows max/mean) | rank step ms (min / mean / max) | "
              "projected masked tok/s | per GPU | efficiency vs N = 1 |")
        print("|---|---|---|---|---|---|---|")
        ref = None
        for n in (1, 2, 4, 8):
            g = dict(base)
            if scaling == "weak":
                g["tasks"] = base["tasks"] * n
            rows, times = [], []
            for r in range(n):
                sh = synth.make_shard(g, rank=r, world=n, seed=2603 + base["index"])
                rows.append(sh.n_active)
                times.append(rank_time(sc, sh, base, pool))
            tot, tmax = sum(rows), max(times)
            val = tot / tmax
            per = val / n
            ref = ref if ref is not None else per
            print(f"| {n} | {tot} | {max(rows) / np.mean(rows):.3f} | {min(times) * 1e3:.1f} / "
                  f"{np.mean(times) * 1e3:.1f} / {tmax * 1e3:.1f} | {val / 1e6:.2f} M | {per / 1e6:.2f} M | "
                  f"{per / ref:.3f} |", flush=True)
        print()
    sc.close()


if __name__ == "__main__":
    main()
