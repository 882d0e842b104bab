# compute-sanitizer over every kernel (scripts/sanitize_kernels.py) + the racecheck repro of the
# warp-specialised ring protocol (scripts/racecheck_repro.cu, prebuilt into build/).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_kernels.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
for v in split self split2; do
  timeout 300 compute-sanitizer --tool racecheck build/racecheck_repro $v > gpurun_out/racecheck_repro_$v.log 2>&1
  echo "repro $v rc=$?"; tail -2 gpurun_out/racecheck_repro_$v.log
done
