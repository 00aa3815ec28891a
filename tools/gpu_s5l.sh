# session 5l: final guard: full GPU suite + smoke + default bench on the final library
set -x
OUT=gpurun_out/s5l; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -x -q --durations=5 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; tail -n 10 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -n 1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_default.log 2>&1; tail -n 1 $OUT/bench_default.log | cut -c1-1200
echo done
