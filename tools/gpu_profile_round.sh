# launch list, per-step DRAM traffic, one full capture of the step kernel
CMD="python bench.py --steps 6 --warmup 3 --no-cpu"
$CMD > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"fast_kernel|deep_kernel" --csv --log-file gpurun_out/traffic.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fast_kernel -s 4 -c 1 -o gpurun_out/prof_fast_kernel $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:deep_kernel -s 4 -c 1 -o gpurun_out/prof_deep_kernel $CMD > /dev/null 2>&1
python tools/launches.py gpurun_out/launches.csv
python tools/metrics_csv.py gpurun_out/traffic.csv
