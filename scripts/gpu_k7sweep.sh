# K7 launch-configuration sweep with the tuning build (PRORL_K7_CONFIG), V = 32 000 / 65 536 / 151 936 bf16.
for V in 32000 65536 151936; do
 for cfg in w16u4096g4 w16u4096g2 w16u2048g2 w16u4096 w16u2048 w24u2048 w12u4096; do
  echo -n "$cfg "; PRORL_HOTPATH_LIB=build/variant/tuning/libprorl_hotpath.so PRORL_K7_CONFIG=$cfg timeout 120 python scripts/k7_probe.py --vocab $V --bufs 3 | head -1
 done
done
