# session 5f: run-to-run variation of the C4 step (same build): copy-bandwidth probe, clocks/power/temperature around each run
set -x
OUT=gpurun_out/s5f; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parallel.py -m gpu -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; tail -n 3 $OUT/pytest.log
timeout 600 python -m pytest tests/test_gpu_fullscale.py -m gpu -q -x -p no:cacheprovider -k "single_step" > $OUT/pytest_fs.log 2>&1; tail -n 3 $OUT/pytest_fs.log
probe() {
python - <<'PY'
import torch, time
a = torch.empty(1 << 30, dtype=torch.uint8, device="cuda"); b = torch.empty_like(a)
best = 0
for _ in range(10):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); b.copy_(a); e1.record(); e1.synchronize()
    best = max(best, 2 * a.numel() / (e0.elapsed_time(e1) * 1e-3) / 1e9)
print("copy GB/s %.0f" % best)
PY
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv,noheader
}
for i in 1 2 3 4 5 6; do
  hs=$((i % 2))
  probe >> $OUT/runs.txt 2>&1
  PYTHONHASHSEED=$hs timeout 600 python bench.py --workload c4 --steps 60 --warmup 5 --no-cpu 2>/dev/null | tail -n 1 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print('hashseed $hs ms %.4f min %.4f max %.4f e2e %.3g clocks %s' % (d['ms_per_step'], d['extra']['step_ms_min'], d['extra']['step_ms_max'], d['e2e']['value'], d['clocks']))" >> $OUT/runs.txt
done
cat $OUT/runs.txt
bash tools/gpu_ab_build.sh s5f "" "HOT_RHO32=0" "c4" 2
echo done
