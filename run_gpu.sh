# usage: bash run_gpu.sh TAG [tests|bench|ncu|full]...
TAG=$1; shift
for what in "$@"; do
case $what in
tests) timeout 900 python -m pytest tests -m gpu -q --timeout 180 -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.txt 2>&1; tail -4 gpurun_out/gpu_tests_$TAG.txt ;;
smoke) timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.txt 2>&1; tail -2 gpurun_out/smoke_$TAG.txt ;;
bench) timeout 900 python bench.py > gpurun_out/bench_$TAG.txt 2>&1; tail -3 gpurun_out/bench_$TAG.txt ;;
ncu) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --layers 2 --prompt 2048 --decode 8 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_$TAG.log 2>&1; tail -1 gpurun_out/ncu_launch_$TAG.log ;;
full) ARGS="--layers 2 --prompt 2048 --decode 8 --steps 1 --warmup 1 --no-e2e --no-cpu"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv1d_silu -s 0 -c 1 -o gpurun_out/conv_$TAG python bench.py $ARGS > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_step -s 2 -c 1 -o gpurun_out/dstep_$TAG python bench.py $ARGS > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 8 -c 1 -o gpurun_out/dtproj_$TAG python bench.py $ARGS > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 0 -c 1 -o gpurun_out/decinproj_$TAG python bench.py $ARGS > /dev/null 2>&1
  ls gpurun_out/*$TAG* ;;
micro) timeout 600 python scripts/gemm_micro.py > gpurun_out/micro_$TAG.txt 2>&1; cat gpurun_out/micro_$TAG.txt ;;
scanmicro) for v in "1 4" "2 0" "2 2" "2 4" "2 6"; do set -- $v; SSM_SCAN_VERSION=$1 SSM_SCAN_NPOLY=$2 timeout 120 python scripts/scan_micro.py; done > gpurun_out/scanmicro_$TAG.txt 2>&1; cat gpurun_out/scanmicro_$TAG.txt ;;
esac
done
