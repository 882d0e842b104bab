"""C5-style vocabulary sweep of the logits-streaming kernels on one B200:
K2+K4 (forward + loss), K5 (backward) and K7 (training pass) at V in
{32 000 ... 262 144}, bf16 (and fp32 at 32 000), ~5 GB of logits per launch.
Prints a markdown table (algorithmic GB/s and % of the measured copy peak).
    python scripts/vocab_sweep.py > profiles/r01_vocab_sweep.md"""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2603_18815_b200.hotpath import Scorer  # noqa: E402

peak = 6547.2
try:
    peak = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
except Exception:
    pass
sc = Scorer(0)


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


print(f"| V | dtype | rows | K2+K4 GB/s (% peak) | K5 GB/s (% peak) | K7 GB/s (% peak) | K7 vs K2+K4->K5 |")
print("|---|---|---|---|---|---|---|")
for V, dt in [(32000, torch.float32), (32000, torch.bfloat16), (65536, torch.bfloat16), (131072, torch.bfloat16),
              (151936, torch.bfloat16), (262144, torch.bfloat16)]:
    es = 2 if dt == torch.bfloat16 else 4
    n = int(5.0e9 // (V * es))
    g = torch.Generator(device="cuda").manual_seed(V)
    x = torch.empty((n, V), dtype=dt, device="cuda")
    gout = torch.empty_like(x)
    t = torch.randint(0, V, (n,), device="cuda", dtype=torch.int32, generator=g)
    old = -0.05 - 2.9 * torch.rand(n, device="cuda", generator=g)
    sc.gen_logits(x, n, 0, t, old, seed=3, sigma=2.0)
    adv = torch.randn(64, device="cuda", generator=g, dtype=torch.float64)
    seq = torch.randint(0, 64, (n,), device="cuda", dtype=torch.int32, generator=g)
    turn = torch.randint(0, 30, (n,), device="cuda", dtype=torch.int16, generator=g)
    lp, _ = sc.logprob_entropy(x, t)
    ms2 = timed(lambda: sc.score_rows(x, t, old, adv, seq, turn))
    ms5 = timed(lambda: sc.logits_grad(x, t, lp, old, adv, seq, float(n), grad=gout))
    ms7 = timed(lambda: sc.score_grad(x, t, old, adv, seq, turn, float(n), grad=gout, want_rows=False))
    b2, b5 = n * (V * es + 26), n * (2 * V * es + 26)
    f = lambda b, ms: f"{b / ms / 1e6:.0f} ({100 * b / ms / 1e6 / peak:.0f} %)"  # noqa: E731
    print(f"| {V} | {'bf16' if es == 2 else 'fp32'} | {n} | {f(b2, ms2)} | {f(b5, ms5)} | {f(b5, ms7)} | "
          f"{(ms2 + ms5) / ms7:.2f}x |", flush=True)
    del x, gout
    torch.cuda.empty_cache()
print(f"\nPeak: {peak:.0f} GB/s (MEASURED_PEAKS.json hbm_gbs, copy test). Algorithmic bytes: K2+K4 V*esz+26 per row; "
      f"K5 and K7 2*V*esz+26 per row (read + write).")
