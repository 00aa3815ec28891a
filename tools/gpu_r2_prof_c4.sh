# round 2 first look: box facts, C3/C4 bench lines, C4 launch list + traffic,
# full capture of the C4 hot kernel
set -x
mkdir -p gpurun_out/r2d
(nproc; free -g; nvidia-smi -L) > gpurun_out/r2d/box.txt 2>&1
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu > gpurun_out/r2d/bench_c4.log 2>&1
timeout 600 python bench.py --workload c3 --steps 20 --warmup 3 --no-cpu > gpurun_out/r2d/bench_c3.log 2>&1
timeout 600 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > gpurun_out/r2d/plain_c4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'fast_kernel|deep_kernel' -s 6 -c 6 --csv --log-file gpurun_out/r2d/traffic_c4.csv \
  python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > gpurun_out/r2d/ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'fast_kernel|deep_kernel' -s 6 -c 2 \
  -o gpurun_out/r2d/full_c4 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > gpurun_out/r2d/ncu2.log 2>&1
echo done
