"""A/B of K6 launch modes inside the whole step (prorl_score_host with a
hidden-state source, C2 shard): device ms per step. Run one mode per process:
    PRORL_K6_PAIR=0|1 [PRORL_K6_CHUNKS=n] python scripts/k6_step_ab.py [micro-batch rows]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_18815_b200 import synth  # noqa: E402
from paper_2603_18815_b200.hotpath import ScoreConfig, Scorer  # noqa: E402

sc = Scorer(0)
sh = synth.make_shard("c2", seed=2604)
host = sh.batch.pinned()
d, V = 2560, 151936
mb = int(sys.argv[1]) if len(sys.argv) > 1 else 16576
H = torch.randn(mb, d, device="cuda").to(torch.bfloat16)
W = (torch.randn(V, d, device="cuda") * (2.0 / d ** 0.5)).to(torch.bfloat16)
cfg = ScoreConfig(vocab=V, dtype="bf16", microbatch_rows=mb)
fn = lambda row0, n, rows, seq, cu: H[:n]  # noqa: E731
sc.score_host_lmhead(host, cfg, fn, W)
ms = []
for _ in range(3):
    _, tm = sc.score_host_lmhead(host, cfg, fn, W)
    ms.append(float(tm[1] + tm[2] + tm[3]))
print(f"mb {mb}  step device ms {np.median(ms):.1f}  ({sh.n_active / (np.median(ms) / 1e3) / 1e6:.3f} M masked tok/s)")
