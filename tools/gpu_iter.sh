# one iteration on the GPU box: parity tests, C4/C2/C5 bench lines, launch
# list + DRAM traffic of the C4 step kernels: bash tools/gpu_iter.sh OUT [full]
set -x
OUT=gpurun_out/${1:-it}
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parallel.py -m gpu -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1
tail -5 $OUT/pytest.log
for w in c4 c2 c3; do
timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu > $OUT/bench_$w.log 2>&1
tail -1 $OUT/bench_$w.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$w', d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'hot_kernel|deep_kernel' -s 6 -c 6 --csv --log-file $OUT/traffic_c4.csv \
  python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > $OUT/ncu1.log 2>&1
python tools/traffic_json.py $OUT/traffic_c4.csv $OUT/traffic_c4.json | head -30
if [ "$2" = "full" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'hot_kernel|deep_kernel' -s 6 -c 2 \
  -o $OUT/full_c4 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > $OUT/ncu2.log 2>&1
fi
echo iter done
