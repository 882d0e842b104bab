mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rf ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -25 gpurun_out/pytest_gpu.log
