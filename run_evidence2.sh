# Final round-1 evidence: gpu tests, smoke, default bench (+ reference arm), other configs, launch list,
# ncu full reports of the dominant decode kernel and the scan, per-kernel roofline table
TAG=$1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.txt 2>&1; tail -2 gpurun_out/gpu_tests_$TAG.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.txt 2>&1; tail -1 gpurun_out/smoke_$TAG.txt
timeout 900 python bench.py > gpurun_out/bench_$TAG.txt 2>&1; tail -1 gpurun_out/bench_$TAG.txt | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$TAG.txt 2>&1; tail -1 gpurun_out/bench_ref_$TAG.txt | cut -c1-200
for c in falcon7b zamba7b mamba2.8b-long; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_${c}_$TAG.txt 2>&1; tail -1 gpurun_out/bench_${c}_$TAG.txt | cut -c1-200
done
timeout 300 python scripts/kernel_rooflines.py --json gpurun_out/rooflines_$TAG.json > gpurun_out/rooflines_$TAG.txt 2>&1
ARGS="--layers 2 --prompt 2048 --decode 8 --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/decinproj_$TAG python bench.py --layers 2 --prompt 256 --decode 8 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_step -s 4 -c 1 -o gpurun_out/dstep_$TAG python bench.py --layers 2 --prompt 256 --decode 8 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 2 -c 1 -o gpurun_out/scan_$TAG python bench.py $ARGS > /dev/null 2>&1
ls gpurun_out/*$TAG*
