# session 5b: new evaluation test, HOT_PIPE A/B (3 rounds), bench lines + ncu traffic for c2/c3/c5
set -x
OUT=gpurun_out/s5b; mkdir -p $OUT
timeout 600 python -m pytest tests/test_evaluation.py -m gpu -q -x -p no:cacheprovider > $OUT/pytest_eval.log 2>&1; tail -5 $OUT/pytest_eval.log
timeout 300 python -c "
from paper_1705_09339_b200.evaluation import measure_level_costs
for dt in ('float32','float64'):
    p, s = measure_level_costs(state_dtype=dt, return_seconds=True)
    print(dt, p, (s*1e12).round(2).tolist(), 'ps/pixel')
" > $OUT/level_costs.txt 2>&1; cat $OUT/level_costs.txt
bash tools/gpu_ab_build.sh s5b "" "HOT_PIPE=0" "c4" 3
for w in c3 c5 c2; do
  timeout 900 python bench.py --workload $w > $OUT/bench_$w.log 2>&1; tail -1 $OUT/bench_$w.log | cut -c1-600
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'hot_kernel|deep_kernel' -s 6 -c 6 --csv --log-file $OUT/traffic_$w.csv \
    python bench.py --workload $w --steps 2 --warmup 3 --no-cpu > $OUT/ncu_$w.log 2>&1
done
echo done
