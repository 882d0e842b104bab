# K7 cost of the RoundFix sample: base (no correction anywhere) vs first-vector (default), 1/32, 1/64, off.
set -x
for v in 151936 32000; do
  for lib in paper_2603_18815_b200/libprorl_hotpath.so build/variant/k7s32/libprorl_hotpath.so build/variant/k7s64/libprorl_hotpath.so build/variant/k7off/libprorl_hotpath.so; do
    timeout 600 python scripts/lib_ab.py build/ab/base/libprorl_hotpath.so $lib --rounds 4 --vocab $v > gpurun_out/ab.log 2>&1; echo "$lib rc=$?"
    tail -2 gpurun_out/ab.log
  done
done
