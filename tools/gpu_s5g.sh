# session 5g: final round-2 validation: full GPU suite, smoke, default bench, reference arm, C4 launch list + full capture
set -x
OUT=gpurun_out/s5g; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q --durations=8 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; tail -n 14 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -n 1 $OUT/smoke.log
timeout 900 python bench.py --impl reference > $OUT/bench_ref.log 2>&1; tail -n 1 $OUT/bench_ref.log | cut -c1-300
timeout 900 python bench.py > $OUT/bench_default.log 2>&1; tail -n 1 $OUT/bench_default.log
timeout 900 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > $OUT/plain_c4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'hot_kernel|deep_kernel' -s 6 -c 6 --csv --log-file $OUT/traffic_c4.csv \
  python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > $OUT/ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'hot_kernel|deep_kernel' -s 6 -c 2 \
  -o $OUT/full_c4 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > $OUT/ncu2.log 2>&1
timeout 900 python bench.py --workload c5 > $OUT/bench_c5.log 2>&1; tail -n 1 $OUT/bench_c5.log | cut -c1-400
timeout 900 python bench.py --workload c3 > $OUT/bench_c3.log 2>&1; tail -n 1 $OUT/bench_c3.log | cut -c1-400
echo done
