# session 5j: last check of the final library: parity subsets, smoke, default bench, C5 launch list
set -x
OUT=gpurun_out/s5j; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parallel.py tests/test_gpu_multiproc.py tests/test_model_io.py tests/test_evaluation.py tests/test_abi.py -m gpu -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; tail -n 3 $OUT/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -n 1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_default.log 2>&1; tail -n 1 $OUT/bench_default.log | cut -c1-900
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'hot_kernel|deep_kernel' -s 6 -c 6 --csv --log-file $OUT/traffic_c5.csv \
    python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu > $OUT/ncu_c5.log 2>&1; tail -n 2 $OUT/ncu_c5.log | cut -c1-300
echo done
