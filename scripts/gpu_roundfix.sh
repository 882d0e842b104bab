# Round-2 FFMA-rounding correction: A/B against the previous library, device parity report, parity tests.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for v in 151936 32000; do
  timeout 600 python scripts/lib_ab.py build/ab/base/libprorl_hotpath.so paper_2603_18815_b200/libprorl_hotpath.so --rounds 4 --vocab $v > gpurun_out/ab_rf_$v.log 2>&1; echo ab rc=$?
  tail -2 gpurun_out/ab_rf_$v.log
  timeout 600 python scripts/lib_ab.py build/ab/base/libprorl_hotpath.so build/variant/k7s32/libprorl_hotpath.so --rounds 4 --vocab $v --kinds k7 > gpurun_out/ab_rf32_$v.log 2>&1; echo ab32 rc=$?
  tail -1 gpurun_out/ab_rf32_$v.log
done
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_train.py -q --timeout 900 -rf > gpurun_out/pytest_roundfix.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_roundfix.log
timeout 1500 python scripts/parity_dev.py --rows > gpurun_out/parity_dev.log 2>&1; echo parity rc=$?
tail -2 gpurun_out/parity_dev.log
