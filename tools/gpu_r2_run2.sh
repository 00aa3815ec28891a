# whole GPU suite (no -x) + C4 launch list / traffic / full capture of the step kernels
set -x
mkdir -p gpurun_out/r2d
timeout 1500 python -m pytest tests -m gpu -q --durations=15 -p no:cacheprovider > gpurun_out/r2d/pytest_gpu.log 2>&1
tail -30 gpurun_out/r2d/pytest_gpu.log
bash tools/gpu_r2_prof_c4.sh
