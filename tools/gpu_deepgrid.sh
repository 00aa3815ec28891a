for n in 8 4 2 1; do
  echo "== $n"
  COG_DEEP_CTAS_PER_SM=$n ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"deep_kernel" --csv --log-file gpurun_out/dg.csv python bench.py --steps 6 --warmup 3 --no-cpu > /dev/null 2>&1
  python tools/metrics_csv.py gpurun_out/dg.csv | grep time
  COG_DEEP_CTAS_PER_SM=$n python bench.py --steps 40 --warmup 5 --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('  ms', d['ms_per_step'])"
done
