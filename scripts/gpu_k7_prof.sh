# K7 evidence: timing (k7_probe) and one ncu --set full capture with source of k_train at V = 151 936.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python scripts/k7_probe.py --bufs 3 --reps 20 > gpurun_out/k7_probe.log 2>&1; echo probe rc=$?
cat gpurun_out/k7_probe.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_train -s 2 -c 1 -o gpurun_out/k7_cur \
  python scripts/k7_probe.py --reps 2 > gpurun_out/k7_ncu.log 2>&1; echo ncu rc=$?
ls -la gpurun_out/*.ncu-rep
