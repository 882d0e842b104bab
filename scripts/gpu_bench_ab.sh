# Whole-bench A/B of library builds, alternating on one box (args: library paths).
for r in 1 2; do
  for lib in "$@"; do
    PRORL_HOTPATH_LIB=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-backward > gpurun_out/bab.log 2>&1
    echo "$r $lib $(tail -1 gpurun_out/bab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,3), round(d["ms_per_step"],2), round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"])')"
  done
done
