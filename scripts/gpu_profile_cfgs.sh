# ncu --set full of k_score for several launch configs (1 GPU).
mkdir -p gpurun_out
for cfg in ${CFGS:-w16s2c4096g2 w16s2c4096g4}; do
  PRORL_K2_CONFIG=$cfg ncu --set full --clock-control none --import-source on -k regex:k_score -s 3 -c 1 \
     -o gpurun_out/prof_$cfg python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof_$cfg.log 2>&1
  echo "$cfg rc=$?"
done
