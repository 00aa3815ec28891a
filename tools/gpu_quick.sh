# quick GPU check: parity tests (not the full-scale ones) + C4/C2 bench lines
# for the default step kernel and, for an A/B, the variant named in $2
set -x
OUT=gpurun_out/${1:-q}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parallel.py -m gpu -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1
tail -5 $OUT/pytest.log
for v in auto ${2:-}; do
for w in c4 c2; do
timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu --variant $v > $OUT/bench_${w}_$v.log 2>&1
tail -1 $OUT/bench_${w}_$v.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$w $v', d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'])"
done
done
