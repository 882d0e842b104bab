# ncu --set full (with source) of one K7 launch of the in-tree library at V = ${V:-151936}
set -x
for V in ${VOCABS:-151936}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_train -s 2 -c 1 -o gpurun_out/k7_new_$V \
  python scripts/k7_probe.py --reps 2 --vocab $V > gpurun_out/k7_ncu_$V.log 2>&1; echo ncu rc=$?
done
ls -la gpurun_out/*.ncu-rep
