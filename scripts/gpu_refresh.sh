mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r_tests.log 2>&1; echo tests; tail -1 gpurun_out/r_tests.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_kernels.py > gpurun_out/r_memcheck.log 2>&1; echo memcheck rc=$?; tail -2 gpurun_out/r_memcheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python scripts/sanitize_kernels.py > gpurun_out/r_synccheck.log 2>&1; echo synccheck rc=$?; tail -2 gpurun_out/r_synccheck.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r_launches_bench.log 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_train -s 2 -c 1 -o gpurun_out/r_prof_k_train python scripts/k7_probe.py --reps 2 --bufs 2 > gpurun_out/r_prof_k7.log 2>&1; echo k7 rc=$?
for i in 1 2; do python bench.py > gpurun_out/r_bench$i.log 2> gpurun_out/r_bench$i.err; echo bench$i rc=$?; done
