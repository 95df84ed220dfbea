set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 180 -p no:cacheprovider > gpurun_out/gpu_tests_2.txt 2>&1
tail -15 gpurun_out/gpu_tests_2.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_2.txt 2>&1; tail -3 gpurun_out/smoke_2.txt
timeout 600 python bench.py --layers 4 --prompt 256 --decode 8 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_small_2.txt 2>&1; tail -5 gpurun_out/bench_small_2.txt
timeout 900 python bench.py > gpurun_out/bench_full_2.txt 2>&1; tail -5 gpurun_out/bench_full_2.txt
