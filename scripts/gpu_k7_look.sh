# K7 experiment: lookahead of the next row's first pieces ahead of the pass-B re-streams (look3 / look5) vs none.
for L in 5 3; do
  PRORL_HOTPATH_LIB=build/variant/look$L/libprorl_hotpath.so timeout 600 python -m pytest tests/test_gpu_train.py -x -q --timeout 300 > gpurun_out/look$L.test.log 2>&1; echo "look$L tests rc=$?"; tail -2 gpurun_out/look$L.test.log
done
for v in 151936 262144 131072 65536; do
  for L in 5 3; do
    timeout 600 python scripts/lib_ab.py paper_2603_18815_b200/libprorl_hotpath.so build/variant/look$L/libprorl_hotpath.so --rounds 4 --vocab $v --kinds k7 > gpurun_out/ab.log 2>&1; echo "look$L rc=$?"
    tail -1 gpurun_out/ab.log
  done
done
