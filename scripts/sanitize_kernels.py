"""Small invocations of every kernel, for compute-sanitizer (memcheck /
racecheck / synccheck):  compute-sanitizer --tool memcheck python scripts/sanitize_kernels.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_18815_b200 import synth  # noqa: E402
from paper_2603_18815_b200.hotpath import LossConfig, ScoreConfig, Scorer  # noqa: E402

dev = torch.device("cuda:0")
s = Scorer(0)
sh = synth.make_shard("c1", seed=99)
b = sh.batch
# K1 + K3 + K2/K4 fused + slab reduce, whole step (fp32 logits, V=32000)
cfg = ScoreConfig(vocab=32000, dtype="fp32", microbatch_rows=1000)
pool = [torch.empty((1000, 32000), dtype=torch.float32, device=dev)]
s.score_host(b.pinned(), cfg, pool, fill=True, seed=3)
# bf16 K2 with odd vocab / padded stride / row indirection, K4 standalone, K5, K6
V, n = 1003, 70
x = torch.empty((n, V + 5), dtype=torch.bfloat16, device=dev)
t = torch.randint(0, V, (n,), dtype=torch.int32, device=dev)
old = torch.full((n,), -1.2, device=dev)
s.gen_logits(x, n, 0, t, old, vocab=V)
rows = torch.randperm(n, device=dev).to(torch.int32)
lp, ent = s.logprob_entropy(x, t, rows=rows, vocab=V)
adv = torch.randn(8, device=dev, dtype=torch.float64)
seq = torch.randint(0, 8, (n,), dtype=torch.int32, device=dev)
turn = torch.randint(0, 70, (n,), dtype=torch.int16, device=dev)
s.clipped_loss(lp, ent, old, adv, seq, turn, cfg=LossConfig(kl_coef=1e-4), ref_lp=lp + 0.1)
s.score_rows(x, t, old, adv, seq, turn, rows=rows, vocab=V)
s.logits_grad(x, t, lp, old, adv, seq, float(n), rows=rows, vocab=V)
# K7 one-pass training step: odd vocab / padded stride / row indirection / in place (two row groups),
# and a large-row bf16 case (one row group, rows longer than the shared-memory ring)
s.score_grad(x, t, old, adv, seq, turn, float(n), rows=rows, vocab=V, grad=x, want_dlogp=True)
xl = torch.empty((24, 151936), dtype=torch.bfloat16, device=dev)
tl = torch.randint(0, 151936, (24,), dtype=torch.int32, device=dev)
s.gen_logits(xl, 24, 0, tl, old[:24])
s.score_grad(xl, tl, old[:24], adv, seq[:24], turn[:24], 24.0, cfg=LossConfig(kl_coef=1e-4), ref_lp=old[:24] + 0.1)
# K7 inside the whole step (training mode, gradient pool)
gpool = [torch.empty_like(pool[0])]
s.score_host(b.pinned(), cfg, pool, fill=True, seed=3, train=True, grad_pool=gpool)
H = torch.randn(200, 256, device=dev).to(torch.bfloat16)
W = (torch.randn(4099, 256, device=dev) * 0.1).to(torch.bfloat16)
s.lmhead_logprob(H, W, torch.randint(0, 4099, (200,), dtype=torch.int32, device=dev))
# K6 with more 256-row tiles than CTA pairs (75 > 74): the paced multi-wave schedule
H2 = torch.randn(19200, 256, device=dev).to(torch.bfloat16)
s.lmhead_logprob(H2, W, torch.randint(0, 4099, (19200,), dtype=torch.int32, device=dev))
torch.cuda.synchronize()
print("sanitize workload done")
