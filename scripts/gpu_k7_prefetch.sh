# K7 experiment: L2 prefetch of the next row (pf1: at the row's pass-B start, pf2: at its pass-A start) vs none.
for v in 151936 262144 65536; do
  for lib in build/variant/pf1/libprorl_hotpath.so build/variant/pf2/libprorl_hotpath.so; do
    timeout 600 python scripts/lib_ab.py paper_2603_18815_b200/libprorl_hotpath.so $lib --rounds 4 --vocab $v --kinds k7 > gpurun_out/ab.log 2>&1; echo "$lib rc=$?"
    tail -1 gpurun_out/ab.log
  done
done
