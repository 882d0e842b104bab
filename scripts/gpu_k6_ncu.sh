# ncu --set full of one K6 launch (k_lmhead2) and of the cuBLAS GEMM of the unfused path, same shape (16 384 x 2 560 x 151 936)
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lmhead2 -s 1 -c 1 -o gpurun_out/k6_r02 \
  python scripts/k6_probe.py --reps 2 > gpurun_out/k6_ncu.log 2>&1; echo ncu k6 rc=$?
cat > /tmp/gemm.py <<'PY'
import torch
n, d, V = 16384, 2560, 151936
H = torch.randn(n, d, device="cuda").to(torch.bfloat16)
W = (torch.randn(V, d, device="cuda") * (2.0 / d ** 0.5)).to(torch.bfloat16)
out = torch.empty((n, V), dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    torch.matmul(H, W.T, out=out)
torch.cuda.synchronize()
PY
timeout 900 ncu --set full --clock-control none -k regex:nvjet -s 2 -c 1 -o gpurun_out/gemm_r02 python /tmp/gemm.py > gpurun_out/gemm_ncu.log 2>&1; echo ncu gemm rc=$?
ls -la gpurun_out/*.ncu-rep
