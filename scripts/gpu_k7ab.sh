# K7/K2 A/B of the round-1 library against the working tree, then the K7 GPU tests.
set -x
for V in 151936 32000 65536 262144; do timeout 300 python scripts/lib_ab.py build/variant/r01/libprorl_hotpath.so paper_2603_18815_b200/libprorl_hotpath.so --vocab $V; done
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_fullsize.py tests/test_cpp_facade.py tests/test_reference_seam.py -q -k "train or score_grad or cpp or seam" > gpurun_out/pytest_train.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest_train.log
