# K2 launch-config sweep + GPU tests (run under gpurun, 1 GPU).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
for cfg in ${CFGS:-w16s2c4096g2 w16s2c4096g4 w12s3c4096g2 w8s3c8192g4}; do
  PRORL_K2_CONFIG=$cfg timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_$cfg.log 2>&1
  echo "$cfg $(python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$cfg.log').read().strip().splitlines()[-1]); print(round(d['value']/1e6,3), 'Mtok/s', round(d['roofline']['achieved']), 'GB/s', round(d['roofline']['frac'],4), d['clocks'])")"
done
