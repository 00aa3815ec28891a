# session 5h: CTA shape / register cap A/B for the hot kernel (build flags only)
set -x
bash tools/gpu_ab_build.sh s5h "" "HOT_TPB=1 COG_HOT_MINB=27" "c4" 2
bash tools/gpu_ab_build.sh s5h "HOT_TPB=3 COG_HOT_MINB=27" "HOT_TPB=1" "c4" 1
bash tools/gpu_ab_build.sh s5h "" "HOT_TPB=1 COG_HOT_MINB=27" "c5 c2" 1
echo done
