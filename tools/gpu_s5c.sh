# session 5c: P2P mailbox tests, two-ended worklist parity, cost-attribution builds, C5/C4 training profile
set -x
OUT=gpurun_out/s5c; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parallel.py tests/test_gpu_multiproc.py tests/test_gpu_parity.py tests/test_abi.py -m gpu -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; tail -8 $OUT/pytest.log
timeout 600 python -m pytest tests/test_gpu_fullscale.py -m gpu -q -x -p no:cacheprovider -k "single_step or c2_whole" > $OUT/pytest_fs.log 2>&1; tail -3 $OUT/pytest_fs.log
timeout 600 python tools/train_profile.py 5 > $OUT/train_c5.txt 2>&1; head -45 $OUT/train_c5.txt
timeout 600 python tools/train_profile.py 4 > $OUT/train_c4.txt 2>&1; head -30 $OUT/train_c4.txt
bash tools/gpu_ab_build.sh s5c "" "HOT_EXP_NORED=1" "c4" 1
bash tools/gpu_ab_build.sh s5c "HOT_EXP_LINEAR=1" "HOT_EXP_NOMODES=1" "c4" 1
bash tools/gpu_ab_build.sh s5c "HOT_EXP_NOCONF=1" "HOT_EXP_NORED=1 HOT_EXP_LINEAR=1 HOT_EXP_NOMODES=1 HOT_EXP_NOCONF=1" "c4" 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'hot_kernel|deep_kernel' -s 6 -c 6 --csv --log-file $OUT/traffic_c4.csv \
    python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > $OUT/ncu_c4.log 2>&1
echo done
