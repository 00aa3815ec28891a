# round-end evidence: GPU tests, smoke, profiles (launch list, traffic, full
# captures), then the bench lines of every workload and the reference arm
set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
bash tools/gpu_profile_round.sh > gpurun_out/profile_round.log 2>&1
bash tools/gpu_bench_all.sh
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log
