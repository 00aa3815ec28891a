# full GPU suite + smoke + the default bench line (with cpu_baseline) +
# deep-kernel occupancy A/B
set -x
OUT=gpurun_out/${1:-full}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q --durations=10 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
tail -12 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_default.log 2>&1; tail -1 $OUT/bench_default.log
bash tools/gpu_ab_build.sh ${1:-full} "" "DEEP_MINB=3" "c4 c5" 1
