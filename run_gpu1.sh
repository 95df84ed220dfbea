nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q --timeout 180 -p no:cacheprovider 2>&1 | tail -60 > gpurun_out/gpu_tests_1.txt
cat gpurun_out/gpu_tests_1.txt | tail -40
