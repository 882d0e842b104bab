# K7 probe across the row-size classes (1, 2, 4 row groups) + the K7 GPU tests.
set -x
for V in 151936 32000 65536 262144; do timeout 300 python scripts/k7_probe.py --vocab $V --bufs 3; done
timeout 300 python scripts/k7_probe.py --vocab 32000 --fp32 --bufs 3
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_fullsize.py tests/test_cpp_facade.py -q -k "train or score_grad or cpp" > gpurun_out/pytest_train.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest_train.log
