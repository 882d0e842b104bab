# K7 A/B of several library builds against a baseline (alternating), after the K7 parity tests.
# usage: LIBS="lib1 lib2 ..." BASE=... VOCABS="..." bash scripts/gpu_k7ab3.sh
set -x
BASE=${BASE:-build/variant/base/libprorl_hotpath.so}
timeout 900 python -m pytest tests/test_gpu_train.py -q -x --timeout 600 > gpurun_out/k7_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/k7_tests.log
for L in ${LIBS:-paper_2603_18815_b200/libprorl_hotpath.so}; do
  for V in ${VOCABS:-151936 32000}; do
    echo "== $L"
    timeout 300 python scripts/lib_ab.py $BASE $L --vocab $V --rounds ${ROUNDS:-4} --kinds k7 2>&1 | tail -1
  done
done
