# K7 with the re-streamed share of each row held in TMEM (default) vs the L2 re-stream (notm build).
timeout 900 python -m pytest tests/test_gpu_train.py -x -q --timeout 600 > gpurun_out/tm_train.log 2>&1; echo "train tests rc=$?"; tail -n 3 gpurun_out/tm_train.log
for v in 151936 131072 200000 65536; do
  timeout 600 python scripts/lib_ab.py build/variant/notm/libprorl_hotpath.so paper_2603_18815_b200/libprorl_hotpath.so --rounds 4 --vocab $v --kinds k7 > gpurun_out/ab.log 2>&1; echo "ab rc=$?"
  tail -n 1 gpurun_out/ab.log
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q --timeout 600 -k "train" > gpurun_out/tm_full.log 2>&1; echo "fullsize train rc=$?"; tail -n 3 gpurun_out/tm_full.log
