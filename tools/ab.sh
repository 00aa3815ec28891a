# A/B: pipelined vs general step kernel on the bench workload (ncu durations)
for mode in pipe general; do
  if [ $mode = general ]; then export COG_NO_PIPE=1; else unset COG_NO_PIPE; fi
  echo "== $mode"
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"step_kernel|pipe_kernel|deep_kernel" --csv --log-file gpurun_out/ab.csv python bench.py --steps 6 --warmup 3 --no-cpu > /dev/null 2>&1
  python tools/launches.py gpurun_out/ab.csv 2>/dev/null | grep -v Fill
  python bench.py --steps 30 --warmup 5 --no-cpu 2>&1 | python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]); print('   bench ms/step', d['ms_per_step'])"
done
