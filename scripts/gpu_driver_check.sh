# What the driver runs at round end: smoke, the GPU suite, bench.py (defaults) and the reference arm.
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench.log | cut -c1-700
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
tail -1 gpurun_out/bench_ref.log | cut -c1-300
