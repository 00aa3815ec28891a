# DRAM bytes + duration per launch of our kernels (one ncu pass)
CMD="python bench.py --steps 6 --warmup 3 --no-cpu"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,smsp__inst_executed.sum \
    --clock-control none -k regex:"step_kernel|deep_kernel" --csv \
    --log-file gpurun_out/mem.csv $CMD > gpurun_out/ncu_mem.log 2>&1
python - <<'PY'
import csv
from collections import defaultdict
rows=[r for r in csv.reader(open('gpurun_out/mem.csv')) if len(r)>5]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
d=defaultdict(lambda: defaultdict(list))
for r in rows[1:]:
    try: d[r[ki][:40]][r[mi]+' '+r[ui]].append(float(r[vi].replace(',','')))
    except: pass
for k,m in d.items():
    print(k)
    for n,v in m.items(): print('   %-55s %12.3f'%(n, sum(v)/len(v)))
PY
