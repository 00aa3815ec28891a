# parity tests + smoke + bench + per-kernel launch times (ncu launch list)
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 30 --warmup 5 --cpu-frames 5 > gpurun_out/bench.log 2>&1
CMD="python bench.py --steps 6 --warmup 3 --no-cpu"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log
python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench.log') if l.startswith('{')][-1]); print('ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'])"
python tools/launches.py gpurun_out/launches.csv
