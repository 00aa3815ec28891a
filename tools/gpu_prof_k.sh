# full ncu capture of one kernel (regex in $1) from a short bench run
K=${1:-lean_kernel}
CMD="python bench.py --steps 6 --warmup 3 --no-cpu"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K \
    -s 4 -c 1 -o gpurun_out/prof_$K $CMD > gpurun_out/ncu_full_$K.log 2>&1
tail -2 gpurun_out/ncu_full_$K.log
