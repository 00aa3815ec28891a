# session 5e: barrier-free atomic union mask: parity + A/B
set -x
OUT=gpurun_out/s5e; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parallel.py tests/test_gpu_multiproc.py -m gpu -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; tail -4 $OUT/pytest.log
timeout 900 python -m pytest tests/test_gpu_fullscale.py -m gpu -q -x -p no:cacheprovider -k "single_step or c2_whole or c5_batch" > $OUT/pytest_fs.log 2>&1; tail -3 $OUT/pytest_fs.log
bash tools/gpu_ab_build.sh s5e "" "HOT_MASK_ATOMIC=0" "c4" 3
bash tools/gpu_ab_build.sh s5e "" "HOT_MASK_ATOMIC=0" "c3 c2" 1
echo done
