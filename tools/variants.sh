# time several builds of the extension on the same workload
for so in build_variants_*.so; do
  echo "== $so"
  COG_LIB=$PWD/$so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu 2>&1 | python -c "import sys,json; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]) if l else {}; print(d.get('ms_per_step'), d.get('extra',{}).get('warm_l2_ms_per_step'), d.get('roofline',{}).get('frac'))"
done
