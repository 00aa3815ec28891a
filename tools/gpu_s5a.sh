# session 5: full GPU suite, smoke, default bench, reference arm
set -x
OUT=gpurun_out/s5a; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q --durations=10 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; tail -15 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_default.log 2>&1; tail -1 $OUT/bench_default.log
timeout 900 python bench.py --impl reference > $OUT/bench_ref.log 2>&1; tail -1 $OUT/bench_ref.log
nproc; free -g | head -2
echo done
