# time several builds of the extension on the same workload (ncu durations)
for so in build_variants_*.so; do
  echo "== $so"
  COG_LIB=$PWD/$so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"step_kernel|pipe_kernel|deep_kernel" --csv --log-file gpurun_out/var.csv python bench.py --steps 6 --warmup 3 --no-cpu > /dev/null 2>&1
  python tools/launches.py gpurun_out/var.csv | grep -v Fill
done
