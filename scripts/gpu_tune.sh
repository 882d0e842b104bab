# K2 launch-config sweep + GPU tests (run under gpurun, 1 GPU).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
for cfg in w16s2c4096 w12s3c4096 w14s3c4096 w8s5c4096; do
  PRORL_K2_CONFIG=$cfg timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_$cfg.log 2>&1
  echo "$cfg $(python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$cfg.log').read().strip().splitlines()[-1]); print(round(d['value']/1e6,3), 'Mtok/s', round(d['roofline']['achieved']), 'GB/s', d['roofline']['frac'], d['clocks'])")"
done
