timeout 1200 bash tools/variants.sh > gpurun_out/variants.log 2>&1
cat gpurun_out/variants.log
bash tools/gpu_prof_k.sh fast_kernel
