"""K7 probe: time the one-pass training kernel (and the two-pass K2+K4 -> K5
sequence) on one C2 micro-batch; run under ncu for the kernel profile.
    python scripts/k7_probe.py [--rows 16576] [--vocab 151936] [--reps 10]"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_18815_b200.hotpath import Scorer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=16576)
ap.add_argument("--vocab", type=int, default=151936)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--fp32", action="store_true")
ap.add_argument("--bufs", type=int, default=1, help="rotate over this many logits buffers (no L2 carry-over)")
a = ap.parse_args()
sc = Scorer(0)
n, V = a.rows, a.vocab
dt = torch.float32 if a.fp32 else torch.bfloat16
xs = [torch.empty((n, V), dtype=dt, device="cuda") for _ in range(a.bufs)]
x = xs[0]
gout = torch.empty_like(x)
g = torch.Generator(device="cuda").manual_seed(7)
t = torch.randint(0, V, (n,), device="cuda", dtype=torch.int32, generator=g)
old = -0.05 - 2.9 * torch.rand(n, device="cuda", generator=g)
for xb in xs:
    sc.gen_logits(xb, n, 0, t, old, seed=3, sigma=2.0)
adv = torch.randn(64, device="cuda", generator=g, dtype=torch.float64)
seq = torch.randint(0, 64, (n,), device="cuda", dtype=torch.int32, generator=g)
turn = torch.randint(0, 30, (n,), device="cuda", dtype=torch.int16, generator=g)


def timed(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


it = [0]


def nxt():
    it[0] += 1
    return xs[it[0] % len(xs)]


ms7 = timed(lambda: sc.score_grad(nxt(), t, old, adv, seq, turn, float(n), grad=gout, want_rows=False))
ms2 = timed(lambda: sc.score_rows(x, t, old, adv, seq, turn))
ms5 = timed(lambda: sc.logits_grad(x, t, old, old, adv, seq, float(n), grad=gout))
bpr = 2 * V * x.element_size() + 30
print(f"V {V}  K7 {ms7:.3f} ms ({n * bpr / ms7 / 1e6:.0f} GB/s)  "
      f"K2+K4 {ms2:.3f} ms  K5 {ms5:.3f} ms  two-pass {ms2 + ms5:.3f} ms  speedup {(ms2 + ms5) / ms7:.2f}")
