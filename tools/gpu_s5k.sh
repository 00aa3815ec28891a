# session 5k: deep kernel item pipeline: parity + A/B
set -x
OUT=gpurun_out/s5k; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parallel.py tests/test_gpu_multiproc.py -m gpu -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; tail -n 3 $OUT/pytest.log
timeout 900 python -m pytest tests/test_gpu_fullscale.py -m gpu -q -x -p no:cacheprovider -k "single_step or c2_whole or c5_batch" > $OUT/pytest_fs.log 2>&1; tail -n 3 $OUT/pytest_fs.log
bash tools/gpu_ab_build.sh s5k "" "DEEP_AHEAD=0" "c4" 2
bash tools/gpu_ab_build.sh s5k "" "DEEP_AHEAD=0" "c5 c2" 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'hot_kernel|deep_kernel' -s 6 -c 6 --csv --log-file $OUT/traffic_c4.csv \
    python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > $OUT/ncu_c4.log 2>&1
echo done
