for so in "" build_variants_*.so; do
  if [ -n "$so" ]; then export COG_LIB=$PWD/$so; else unset COG_LIB; fi
  echo "== ${so:-default}"
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none -k regex:"fast_kernel|deep_kernel" --csv --log-file gpurun_out/abl.csv python bench.py --steps 6 --warmup 3 --no-cpu > /dev/null 2>&1
  python tools/metrics_csv.py gpurun_out/abl.csv | grep -v "^ *[0-9]* x void <unnamed>::deep" 
done
