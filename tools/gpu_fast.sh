timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 1200 bash tools/variants.sh > gpurun_out/variants.log 2>&1
cat gpurun_out/variants.log
