# Round-2 final evidence pass: smoke, GPU suite, device parity report, bench (ours + reference arm),
# k_score ncu capture (traffic, stamped with the SASS digest) and the launch list.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -6 gpurun_out/pytest_gpu.log
timeout 1500 python scripts/parity_dev.py --rows > gpurun_out/parity_dev.log 2>&1; echo parity rc=$?
tail -1 gpurun_out/parity_dev.log | cut -c1-300
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo bench rc=$?
tail -c 1200 gpurun_out/bench_c3.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
tail -c 600 gpurun_out/bench_ref.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_score -s 3 -c 1 -o gpurun_out/prof_k_score_r02f \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-backward > gpurun_out/prof_k_score_r02f.log 2>&1; echo ncu rc=$?
python -c "import bench; print(bench.k_score_stamp())" > gpurun_out/k_score_sass_stamp.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02f.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-backward > gpurun_out/launches_r02f.log 2>&1; echo launches rc=$?
ls -la gpurun_out
