# ncu --set full of one K7 launch from each of two library builds (A/B), V = 151 936 and 32 000.
set -x
for V in 151936 32000; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_train -s 4 -c 1 -o gpurun_out/k7_r01_$V \
  python scripts/lib_ab.py build/variant/r01/libprorl_hotpath.so build/variant/r01/libprorl_hotpath.so --vocab $V --rounds 1 --reps 2 --kinds k7 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_train -s 4 -c 1 -o gpurun_out/k7_r02_$V \
  python scripts/lib_ab.py paper_2603_18815_b200/libprorl_hotpath.so paper_2603_18815_b200/libprorl_hotpath.so --vocab $V --rounds 1 --reps 2 --kinds k7 > /dev/null 2>&1
done
ls -la gpurun_out/*.ncu-rep
