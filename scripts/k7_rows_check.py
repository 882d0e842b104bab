"""Per-row logp / entropy of K2 and K7 vs the fp64 oracle on the same rows
(mean signed error = the systematic residual), for a few vocabularies."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle as O  # noqa: E402
from paper_2603_18815_b200.hotpath import Scorer  # noqa: E402

s = Scorer(0)
for V, n in [(151936, 2048), (262144, 1536), (65536, 4096), (32000, 4096)]:
    rng = np.random.default_rng(V)
    t = rng.integers(0, V, n).astype(np.int32)
    old = (-0.05 - 2.9 * rng.random(n)).astype(np.float32)
    x = torch.empty((n, V), dtype=torch.bfloat16, device="cuda")
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    s.gen_logits(x, n, 12345, dv(t), dv(old), seed=31, sigma=2.0)
    host = O.gen_logits(n, V, 12345, t, old, seed=31, sigma=2.0, dtype="bf16")
    olp, oent = O.logprob_entropy(host, t)
    lp2, ent2 = s.logprob_entropy(x, dv(t))
    adv = dv(rng.normal(0, 1, 8))
    seq = dv(rng.integers(0, 8, n).astype(np.int32))
    turn = dv(np.zeros(n, np.int16))
    _, lp7, ent7, _, _ = s.score_grad(x, dv(t), dv(old), adv, seq, turn, float(n))
    for name, g, o in (("K2 logp", lp2, olp), ("K7 logp", lp7, olp), ("K2 ent", ent2, oent), ("K7 ent", ent7, oent)):
        e = g.cpu().numpy().astype(np.float64) - o
        print(f"V={V} {name}: mean {e.mean():+.3e} rms {np.sqrt((e*e).mean()):.3e} max|e| {np.abs(e).max():.3e}")
