# GPU check used during round 2: smoke, the GPU suite, the full-size parity device run.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rf ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -40 gpurun_out/pytest_gpu.log
if [ -n "${PARITY_DEV:-}" ]; then timeout 900 python scripts/parity_dev.py $PARITY_DEV > gpurun_out/parity_dev.log 2>&1; echo parity rc=$?; tail -5 gpurun_out/parity_dev.log; fi
if [ -n "${BENCH:-}" ]; then timeout 900 python bench.py $BENCH > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -c 3000 gpurun_out/bench.log; fi
