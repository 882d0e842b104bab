import sys, torch
sys.path.insert(0, ".")
from paper_2603_18815_b200.hotpath import Scorer
sc = Scorer(0)
n, V = int(sys.argv[1]), int(sys.argv[2])
x = torch.randn((n, V), device="cuda").to(torch.bfloat16)
t = torch.randint(0, V, (n,), device="cuda", dtype=torch.int32)
old = torch.full((n,), -1.0, device="cuda")
adv = torch.randn(4, device="cuda")
seq = torch.zeros(n, dtype=torch.int32, device="cuda")
turn = torch.zeros(n, dtype=torch.int16, device="cuda")
p, lp, ent, g, dl = sc.score_grad(x, t, old, adv, seq, turn, float(n))
torch.cuda.synchronize()
print("ok", n, V, p[1].item())
