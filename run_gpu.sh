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
decexp) timeout 600 python scripts/decode_gemm_exp.py > gpurun_out/decexp_$TAG.txt 2>&1; cat gpurun_out/decexp_$TAG.txt ;;
benchnopdl) SSM_PDL=0 timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/benchnopdl_$TAG.txt 2>&1; tail -1 gpurun_out/benchnopdl_$TAG.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NOPDL', d['value'], d['ttft_ms'], d['tpot_ms'])" ;;
decprof) timeout 600 python scripts/decode_profile.py > gpurun_out/decprof_$TAG.txt 2>&1; cat gpurun_out/decprof_$TAG.txt ;;
ablate) (for m in 0 8 16 23 31; do SSM_DEBUG_SKIP=$m timeout 120 python scripts/decode_ablation.py; done; SSM_DEBUG_SKIP_NORM=1 timeout 120 python scripts/decode_ablation.py; SSM_DEBUG_SKIP=31 SSM_DEBUG_SKIP_NORM=1 timeout 120 python scripts/decode_ablation.py; SSM_PDL=0 timeout 120 python scripts/decode_ablation.py; SSM_FUSE_DECODE=0 timeout 120 python scripts/decode_ablation.py; echo dstep-fused-in-out_proj; SSM_FUSE_DSTEP=1 timeout 120 python scripts/decode_ablation.py) > gpurun_out/ablate_$TAG.txt 2>&1; cat gpurun_out/ablate_$TAG.txt ;;
dstepfull) ARGS="--layers 2 --prompt 256 --decode 8 --steps 1 --warmup 1 --no-e2e --no-cpu"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_step -s 4 -c 1 -o gpurun_out/dstep_$TAG python bench.py $ARGS > /dev/null 2>&1; ls gpurun_out/dstep_$TAG* ;;
decinfull) ARGS="--layers 2 --prompt 256 --decode 8 --steps 1 --warmup 1 --no-e2e --no-cpu"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 0 -c 1 -o gpurun_out/decinproj_$TAG python bench.py $ARGS > /dev/null 2>&1; ls gpurun_out/decinproj_$TAG* ;;
stream) timeout 300 python scripts/stream_probe.py > gpurun_out/stream_$TAG.txt 2>&1; cat gpurun_out/stream_$TAG.txt ;;
gtrace) (for a in 1 2 4 8; do SSM_GEMM_NACC=$a SSM_GEMM_NOMMA=8 timeout 120 python scripts/gemm_trace.py; done; SSM_GEMM_NOMMA=9 timeout 120 python scripts/gemm_trace.py; SSM_GEMM_NOMMA=8 timeout 120 python scripts/gemm_trace.py 16 2560 5120) > gpurun_out/gtrace_$TAG.txt 2>&1; cat gpurun_out/gtrace_$TAG.txt ;;
benchpdl) SSM_PDL=1 timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/benchpdl_$TAG.txt 2>&1; tail -1 gpurun_out/benchpdl_$TAG.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PDL', d['value'], d['ttft_ms'], d['tpot_ms'])" ;;
testspdl) SSM_PDL=1 timeout 900 python -m pytest tests -m gpu -q --timeout 180 -p no:cacheprovider > gpurun_out/gpu_testspdl_$TAG.txt 2>&1; tail -4 gpurun_out/gpu_testspdl_$TAG.txt ;;
esac
done
