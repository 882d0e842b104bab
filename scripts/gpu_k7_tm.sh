# K7 TMEM-held re-stream share: 2 KB units (tm1) and 4 KB units (tm2) vs the default.
for m in 2; do
  PRORL_HOTPATH_LIB=build/variant/tm$m/libprorl_hotpath.so timeout 600 python -m pytest tests/test_gpu_train.py -x -q --timeout 300 > gpurun_out/tm$m.log 2>&1; echo "tm$m tests rc=$?"; tail -n 1 gpurun_out/tm$m.log
done
for v in 151936 131072; do
  for m in 1 2; do
    timeout 600 python scripts/lib_ab.py paper_2603_18815_b200/libprorl_hotpath.so build/variant/tm$m/libprorl_hotpath.so --rounds 4 --vocab $v --kinds k7 > gpurun_out/ab.log 2>&1; echo "tm$m rc=$?"; tail -n 1 gpurun_out/ab.log
  done
done
