#!/bin/bash
# Build an experimental variant of the library with extra nvcc flags into
# build/variant/<name>/libprorl_hotpath.so, for A/B runs through
# PRORL_HOTPATH_LIB=<that path>. Usage: scripts/build_variant.sh <name> <nvcc flags...>
# The tuning build (every launch configuration, PRORL_K*_ / PRORL_PDL honoured):
#   scripts/build_variant.sh tuning -DPRORL_TUNING
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/build/variant/$name
mkdir -p "$out"
json=$(python -c "from paper_2603_18815_b200 import build as B; print(B.json_include())")
objs=()
for src in pack.cu grpo.cu score.cu grad.cu train.cu lmhead.cu synth.cu capi.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I"$root/include" -I"$root/paper_2603_18815_b200/csrc" -I"$json" "$@" \
    -c "$root/paper_2603_18815_b200/csrc/$src" -o "$out/${src%.*}.o" &
  objs+=("$out/${src%.*}.o")
done
for src in workload.cpp ingest.cpp; do
  g++ -O3 -std=c++17 -fPIC -I"$root/include" -I"$root/paper_2603_18815_b200/csrc" -I"$json" -I/usr/local/cuda/include \
    -c "$root/paper_2603_18815_b200/csrc/$src" -o "$out/${src%.*}.o" &
  objs+=("$out/${src%.*}.o")
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libprorl_hotpath.so" "${objs[@]}" -ldl
echo "$out/libprorl_hotpath.so"
