"""K6 micro-batch sweep: the fused LM head + logprob (K6) against the unfused
path it replaces (cuBLAS bf16 GEMM writing the logits, then K2) at several
row counts, alternating the two arms so clock drift under the power cap hits
both alike. K6 maps one 256-row tile to one CTA pair and walks the whole
vocabulary (one chunk, paced through L2), so a micro-batch of 74 x 256 = 18 944
rows fills all 148 SMs; 16 384 rows leave 10 of the 74 pairs idle.
    python scripts/k6_rows_sweep.py [--rows 16384,18944,37888] [--rounds 3]"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_18815_b200.hotpath import Scorer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", default="16384,18944,37888")
ap.add_argument("--d", type=int, default=2560)
ap.add_argument("--vocab", type=int, default=151936)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--rounds", type=int, default=3)
a = ap.parse_args()
s = Scorer(0)
d, V = a.d, a.vocab
g = torch.Generator(device="cuda").manual_seed(11)
W = (torch.randn(V, d, device="cuda", generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for n in [int(x) for x in a.rows.split(",")]:
    H = torch.randn(n, d, device="cuda", generator=g).to(torch.bfloat16)
    t = torch.randint(0, V, (n,), device="cuda", dtype=torch.int32, generator=g)
    logits = torch.empty((n, V), dtype=torch.bfloat16, device="cuda")

    def fused():
        s.lmhead_logprob(H, W, t)

    def unfused():
        torch.matmul(H, W.T, out=logits)
        s.logprob_entropy(logits, t)

    def gemm():
        torch.matmul(H, W.T, out=logits)

    k6, un, gm = [], [], []
    for r in range(a.rounds):
        for which in ((0, 1, 2) if r % 2 == 0 else (2, 1, 0)):
            ms = timed((fused, unfused, gemm)[which], a.reps)
            (k6, un, gm)[which].append(ms)
    tf = lambda ms: 2.0 * n * d * V / (ms / 1e3) / 1e12  # noqa: E731
    b6, bu, bg = min(k6), min(un), min(gm)
    print(f"rows {n:6d}: K6 {b6:.3f} ms ({tf(b6):.0f} TFLOP/s)  unfused {bu:.3f} ms  (GEMM alone {bg:.3f} ms, "
          f"{tf(bg):.0f} TFLOP/s)  speedup {bu / b6:.3f}  K6 rows/s {n / b6 * 1e3:.3e}  "
          f"all K6 {['%.3f' % v for v in k6]} unfused {['%.3f' % v for v in un]}", flush=True)
    del H, t, logits
    torch.cuda.empty_cache()
