import sys, os, json, torch
sys.path.insert(0, ".")
from paper_2603_18815_b200.hotpath import Scorer
s = Scorer(0)
n, V = 16576, 151936
x = torch.empty((n, V), dtype=torch.bfloat16, device="cuda"); y = torch.empty_like(x)
t = torch.randint(0, V, (n,), dtype=torch.int32, device="cuda")
old = torch.full((n,), -1.2, device="cuda")
s.gen_logits(x, n, 0, t, old)
lp, _ = s.logprob_entropy(x, t)
adv = torch.randn(64, device="cuda", dtype=torch.float64); seq = torch.randint(0, 64, (n,), dtype=torch.int32, device="cuda")
old2 = lp + 0.3 * (torch.rand(n, device="cuda") - 0.5)
for _ in range(2): s.logits_grad(x, t, lp, old2, adv, seq, float(n), grad=y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): s.logits_grad(x, t, lp, old2, adv, seq, float(n), grad=y)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(os.environ.get("PRORL_K5_CONFIG", "default"), f"{ms:.3f} ms", f"{n*(4*V+26)/ms/1e6:.0f} GB/s")
