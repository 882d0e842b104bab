# ncu evidence for the dominant kernel (run under gpurun, 1 GPU).
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_score -s 3 -c 2 -o gpurun_out/prof_k_score \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof_bench.log 2>&1
echo full rc=$?
ls -la gpurun_out
# K6 (tcgen05 LM head) — one launch at the Qwen3-4B shape
cat > /tmp/k6.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2603_18815_b200.hotpath import Scorer
s = Scorer(0)
n, d, V = 16384, 2560, 151936
H = torch.randn(n, d, device="cuda").to(torch.bfloat16)
W = (torch.randn(V, d, device="cuda") * 0.04).to(torch.bfloat16)
t = torch.randint(0, V, (n,), device="cuda", dtype=torch.int32)
for _ in range(2): s.lmhead_logprob(H, W, t)
torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -k regex:k_lmhead -s 1 -c 1 -o gpurun_out/prof_k_lmhead python /tmp/k6.py > gpurun_out/prof_k6.log 2>&1
echo k6 rc=$?
