# session 5n: CTA shape + deep occupancy combination A/B (build flags only)
set -x
bash tools/gpu_ab_build.sh s5n "" "HOT_TPB=3 COG_HOT_MINB=27 DEEP_MINB=3" "c4" 2
bash tools/gpu_ab_build.sh s5n "" "HOT_TPB=3 COG_HOT_MINB=27 DEEP_MINB=3" "c5" 1
echo done
