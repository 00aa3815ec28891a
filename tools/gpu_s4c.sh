set -x
OUT=gpurun_out/s4c; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
bash tools/gpu_ab_build.sh s4c "" "HOT_PIPE=0" "c4" 2
bash tools/gpu_ab_build.sh s4c "HOT_NS=3" "HOT_NS=6" "c4" 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'hot_kernel|deep_kernel' -s 6 -c 2 \
  -o $OUT/full_c4 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > $OUT/ncu2.log 2>&1
echo done
