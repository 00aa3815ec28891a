# launch list + DRAM traffic of the step kernels, and one full capture of
# the hot kernel and the deep kernel: bash tools/gpu_prof_hot.sh OUT [workload]
OUT=gpurun_out/$1; W=${2:-c4}
mkdir -p $OUT
timeout 600 python bench.py --workload $W --steps 2 --warmup 3 --no-cpu > $OUT/plain_$W.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'hot_kernel|fast_kernel|deep_kernel' -s 6 -c 6 --csv --log-file $OUT/traffic_$W.csv \
  python bench.py --workload $W --steps 2 --warmup 3 --no-cpu > $OUT/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'hot_kernel|deep_kernel' -s 6 -c 2 \
  -o $OUT/full_$W python bench.py --workload $W --steps 2 --warmup 3 --no-cpu > $OUT/ncu2.log 2>&1
echo prof done
