"""K6 probe: time the fused LM head + logprob kernel at the Qwen3-4B LM-head
shape and check it against torch (bf16 GEMM -> fp32 logsumexp) on a few rows.
    PRORL_K6_PAIR=0|1 python scripts/k6_probe.py [--rows 16384] [--d 2560] [--vocab 151936]"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_18815_b200.hotpath import Scorer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=16384)
ap.add_argument("--d", type=int, default=2560)
ap.add_argument("--vocab", type=int, default=151936)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
s = Scorer(0)
g = torch.Generator(device="cuda").manual_seed(1)
H = torch.randn(a.rows, a.d, device="cuda", generator=g).to(torch.bfloat16)
W = (torch.randn(a.vocab, a.d, device="cuda", generator=g) * (2.0 / a.d ** 0.5)).to(torch.bfloat16)
t = torch.randint(0, a.vocab, (a.rows,), device="cuda", dtype=torch.int32, generator=g)
lp, ent = s.lmhead_logprob(H, W, t)
torch.cuda.synchronize()
idx = torch.arange(0, a.rows, max(1, a.rows // 64), device="cuda")
x = (H[idx].double() @ W.double().T)
ref_lp = (x.gather(1, t[idx].long()[:, None])[:, 0] - torch.logsumexp(x, 1))
p = torch.softmax(x, 1)
ref_ent = -(p * torch.log_softmax(x, 1)).sum(1)
err_lp = ((lp[idx].double() - ref_lp).abs() / ref_lp.abs().clamp_min(1e-3)).max().item()
err_ent = ((ent[idx].double() - ref_ent).abs() / ref_ent.abs().clamp_min(1e-3)).max().item()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    s.lmhead_logprob(H, W, t)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
tf = 2.0 * a.rows * a.d * a.vocab / (ms / 1e3) / 1e12
print(f"K6 rows {a.rows} d {a.d} V {a.vocab}: {ms:.3f} ms  {tf:.0f} TFLOP/s  max rel err logp {err_lp:.2e} entropy {err_ent:.2e}")
