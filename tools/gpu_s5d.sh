# session 5d: tiled sequential sums (grouping parity + training time), two-ended / deep A/B
set -x
OUT=gpurun_out/s5d; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parallel.py -m gpu -q -x -p no:cacheprovider -k "grouping or kmeans or pooled or mailbox" > $OUT/pytest.log 2>&1; tail -4 $OUT/pytest.log
timeout 600 python tools/train_profile.py 5 > $OUT/train_c5.txt 2>&1; head -12 $OUT/train_c5.txt
timeout 600 python tools/train_profile.py 4 > $OUT/train_c4.txt 2>&1; head -12 $OUT/train_c4.txt
bash tools/gpu_ab_build.sh s5d "" "HOT_TWO_ENDED=0" "c4" 2
bash tools/gpu_ab_build.sh s5d "DEEP_MINB=3" "DEEP_THREADS=128 DEEP_MINB=4" "c4" 1
bash tools/gpu_ab_build.sh s5d "" "HOT_TWO_ENDED=0" "c5" 1
echo done
