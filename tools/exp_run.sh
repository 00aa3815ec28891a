# compare builds: label COG_LIB=... [ENV=...]; ncu durations/traffic + bench ms
run() {  # label, env...
  echo "== $1"; shift
  env "$@" ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"fast_kernel|deep_kernel" --csv --log-file gpurun_out/var.csv python bench.py --steps 6 --warmup 3 --no-cpu > /dev/null 2>&1
  python tools/metrics_csv.py gpurun_out/var.csv
  env "$@" python bench.py --steps 30 --warmup 5 --no-cpu 2>&1 | python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]); print('   bench ms/step %.4f frac %.3f e2e %.3g' % (d['ms_per_step'], d['roofline']['frac'], d['e2e']['value']))"
}
