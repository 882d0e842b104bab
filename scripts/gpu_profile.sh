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
