for v in X=1 COG_LIB=$PWD/build_variants_d64.so X=1 COG_LIB=$PWD/build_variants_d64.so; do
  env $v python bench.py --workload c5 --streams 8 --steps 10 --warmup 3 --no-cpu 2>&1 | python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]); print('c5 $v'[:40].ljust(40), 'ms/step %.4f e2e %.3g' % (d['ms_per_step'], d['e2e']['value']))"
done
