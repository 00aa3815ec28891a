# full ncu capture of kernel $1 using library $2
K=$1; export COG_LIB=$PWD/$2
CMD="python bench.py --steps 6 --warmup 3 --no-cpu"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 4 -c 1 -o gpurun_out/prof_var $CMD > gpurun_out/ncu_var.log 2>&1
tail -1 gpurun_out/ncu_var.log
