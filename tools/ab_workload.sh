# A/B of one workload's ms/step, alternating: bash tools/ab_workload.sh WL "ENV_A" "ENV_B" [rounds] [steps]
W="$1"; A="$2"; B="$3"; R=${4:-2}; S=${5:-20}
for r in $(seq $R); do
  for v in "$A" "$B"; do
    env $v python bench.py --workload $W --steps $S --warmup 3 --no-cpu 2>&1 | python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]); print('$W', '$v'[-24:].ljust(24), 'ms/step %.4f' % d['ms_per_step'])"
  done
done
