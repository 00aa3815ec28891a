COG_KERNEL=vec timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for k in fast vec; do
  echo "== $k"
  COG_KERNEL=$k ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none -k regex:"fast_kernel|vec_kernel|deep_kernel" --csv --log-file gpurun_out/v.csv python bench.py --steps 6 --warmup 3 --no-cpu > /dev/null 2>&1
  python tools/metrics_csv.py gpurun_out/v.csv
  COG_KERNEL=$k python bench.py --steps 30 --warmup 5 --no-cpu 2>&1 | python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]); print('   bench ms/step %.4f frac %.3f e2e %.3g' % (d['ms_per_step'], d['roofline']['frac'], d['e2e']['value']))"
done
