# full GPU test suite + smoke + quick C4/C2 bench lines (no ncu)
set -x
mkdir -p gpurun_out/r2c
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 -p no:cacheprovider > gpurun_out/r2c/pytest_gpu.log 2>&1
tail -30 gpurun_out/r2c/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c/smoke.log 2>&1; tail -2 gpurun_out/r2c/smoke.log
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu > gpurun_out/r2c/bench_c4.log 2>&1; tail -1 gpurun_out/r2c/bench_c4.log
timeout 600 python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu > gpurun_out/r2c/bench_c2.log 2>&1; tail -1 gpurun_out/r2c/bench_c2.log
