# A/B of bench ms/step, alternating: bash tools/ab_bench.sh "ENV_A" "ENV_B" [rounds]
A="$1"; B="$2"; R=${3:-3}
for r in $(seq $R); do
  for v in "$A" "$B"; do
    env $v python bench.py --steps 60 --warmup 5 --no-cpu 2>&1 | python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]); print('$v'.ljust(24), 'ms/step %.4f e2e %.3g' % (d['ms_per_step'], d['e2e']['value']))"
  done
done
