# A/B of build-time tuning macros on the same box:
#   bash tools/gpu_ab_build.sh OUT "DEFS_A" "DEFS_B" [workloads] [rounds]
# DEFS: space-separated NAME=VALUE (empty string = default build)
OUT=gpurun_out/$1; A="$2"; B="$3"; WL=${4:-"c4 c2"}; R=${5:-2}
mkdir -p $OUT
for r in $(seq $R); do
  for v in "$A" "$B"; do
    python -c "import sys; sys.path.insert(0,'.'); from paper_1705_09339_b200 import _lib; _lib.build_extension(defines=tuple('$v'.split()))" || exit 1
    for w in $WL; do
      python bench.py --workload $w --steps 60 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('[$v]'.ljust(28), '$w', 'ms/step %.4f frac %.3f' % (d['ms_per_step'], d['roofline']['frac']))" | tee -a $OUT/ab.txt
    done
  done
done
python -c "import sys; sys.path.insert(0,'.'); from paper_1705_09339_b200 import _lib; _lib.build_extension(force=True)"
