# session 5i: pooled group statistics on the device for mid-size groups: full-scale parity (C3, C5) + C5 training time
set -x
OUT=gpurun_out/s5i; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_fullscale.py -m gpu -q -x -p no:cacheprovider -k "c3_whole or c5_batch or single_step" --durations=5 > $OUT/pytest_fs.log 2>&1; tail -n 9 $OUT/pytest_fs.log
timeout 900 python -m pytest tests/test_gpu_parallel.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; tail -n 3 $OUT/pytest.log
timeout 900 python bench.py --workload c5 > $OUT/bench_c5.log 2>&1; tail -n 1 $OUT/bench_c5.log | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('c5 ms', d['ms_per_step'], 'value', d['value'], 'train_s', d['extra']['train_s'], 'e2e', d['e2e']['value'])"
timeout 900 python bench.py --workload c3 --no-cpu > $OUT/bench_c3.log 2>&1; tail -n 1 $OUT/bench_c3.log | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('c3 ms', d['ms_per_step'], 'value', d['value'], 'train_s', d['extra']['train_s'])"
echo done
