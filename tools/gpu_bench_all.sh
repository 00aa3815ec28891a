nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_c2.log 2>&1; tail -1 gpurun_out/bench_ref_c2.log
timeout 900 python bench.py --workload c3 --steps 30 > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log
timeout 1200 python bench.py --workload c5 --steps 20 --streams 32 > gpurun_out/bench_c5.log 2>&1; tail -2 gpurun_out/bench_c5.log
timeout 1200 python bench.py --workload c4 --steps 20 > gpurun_out/bench_c4.log 2>&1; tail -2 gpurun_out/bench_c4.log
