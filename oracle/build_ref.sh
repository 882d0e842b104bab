#!/usr/bin/env bash
# Build oracle/_ref/libref.so from the UNMODIFIED reference sources under
# /root/reference (read in place, never copied) plus oracle/ref_shim.cpp.
# Test infrastructure only. Needs g++ (C++20) and nlohmann/json 3.11.3, which
# this image carries under the venv's cudnn_frontend third-party tree.
# Exits 0 without building when /root/reference is absent (GPU box).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${PRORL_REFERENCE:-/root/reference}/proj"
OUT="$HERE/_ref"
if [ ! -d "$REF" ]; then
  echo "build_ref: $REF absent; skipping (prebuilt oracle/_ref is used if present)"
  exit 0
fi
JSON_DIR="${PRORL_JSON_DIR:-}"
if [ -z "$JSON_DIR" ]; then
  JSON_DIR="$(python3 - <<'EOF'
import glob, os, site, sys
cands = []
for sp in site.getsitepackages() + [site.getusersitepackages()]:
    cands += glob.glob(os.path.join(sp, "include", "cudnn_frontend", "thirdparty", "nlohmann"))
print(cands[0] if cands else "")
EOF
)"
fi
if [ -z "$JSON_DIR" ] || [ ! -f "$JSON_DIR/json.hpp" ]; then
  echo "build_ref: json.hpp not found; cannot build the reference oracle" >&2
  exit 1
fi
mkdir -p "$OUT/obj"
CXX="${CXX:-g++}"
FLAGS=(-std=c++20 -O2 -fPIC -I"$REF/include" -I"$JSON_DIR")
for src in src/trainer/harness.cpp src/trainer/workload.cpp src/mock/policy.cpp src/handlers.cpp \
           src/sandbox/build_cache.cpp src/sandbox/framing.cpp src/sandbox/proc.cpp src/sandbox/runtime.cpp; do
  "$CXX" "${FLAGS[@]}" -c "$REF/$src" -o "$OUT/obj/$(basename "$src" .cpp).o"
done
"$CXX" "${FLAGS[@]}" -c "$HERE/ref_shim.cpp" -o "$OUT/obj/ref_shim.o"
"$CXX" -shared -Wl,--no-undefined -o "$OUT/libref.so" "$OUT"/obj/*.o -lpthread
echo "$OUT/libref.so"
