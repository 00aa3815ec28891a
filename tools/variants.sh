# time several builds / kernel choices on the bench workload (ncu durations + bench ms)

run() {  # label, env...
  echo "== $1"; shift
  env "$@" ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"step_kernel|pipe_kernel|deep_kernel|lean_kernel|fast_kernel" --csv --log-file gpurun_out/var.csv python bench.py --steps 6 --warmup 3 --no-cpu > /dev/null 2>&1
  python tools/metrics_csv.py gpurun_out/var.csv
  env "$@" python bench.py --steps 30 --warmup 5 --no-cpu 2>&1 | python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]); print('   bench ms/step %.4f frac %.3f e2e %.3g' % (d['ms_per_step'], d['roofline']['frac'], d['e2e']['value']))"
}
run default X=1
[ -n "$WITH_PIPE" ] && run pipe COG_KERNEL=pipe
[ -n "$WITH_LEAN" ] && run lean COG_KERNEL=lean
[ -n "$WITH_FAST" ] && run fast COG_KERNEL=fast
for so in build_variants_*.so; do run $so COG_LIB=$PWD/$so; done
