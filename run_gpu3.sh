timeout 600 python -m pytest tests -m gpu -q --timeout 180 -p no:cacheprovider -k "virtual" > gpurun_out/gpu_tests_3.txt 2>&1; tail -3 gpurun_out/gpu_tests_3.txt
ARGS="--layers 2 --prompt 2048 --decode 8 --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_3.csv python bench.py $ARGS > gpurun_out/ncu_launch_3.log 2>&1; tail -2 gpurun_out/ncu_launch_3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 2 -c 1 -o gpurun_out/scan_3 python bench.py $ARGS > gpurun_out/ncu_scan_3.log 2>&1; tail -2 gpurun_out/ncu_scan_3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 10 -c 1 -o gpurun_out/gemm_3 python bench.py $ARGS > gpurun_out/ncu_gemm_3.log 2>&1; tail -2 gpurun_out/ncu_gemm_3.log
ls -la gpurun_out
