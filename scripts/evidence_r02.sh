#!/bin/bash
# Round-2 evidence run on one B200 (gpurun): GPU tests, default bench line, reference arm, every
# BASELINE config, ncu launch list of a 2-layer bench, ncu --set full of the top kernels, decode
# timeline.  Everything lands in gpurun_out/ev_*; copy the ones to judge into profiles/.
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/ev_gputest.log 2>&1; tail -2 $O/ev_gputest.log
timeout 900 python bench.py > $O/ev_bench.json 2> $O/ev_bench.err; tail -c 600 $O/ev_bench.json
timeout 900 python bench.py --impl reference > $O/ev_bench_ref.json 2> $O/ev_bench_ref.err
rm -f $O/ev_sweep.jsonl; timeout 2400 python scripts/config_sweep.py $O/ev_sweep.jsonl > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ev_launches.csv \
  python bench.py --steps 2 --warmup 1 --layers 2 --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_stack_kernel -c 1 -o $O/ev_dstack \
  python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_kernel -c 1 -o $O/ev_scan \
  python scripts/prefill_time.py --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -c 1 -o $O/ev_inproj \
  python scripts/prefill_time.py --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:m2_ssd_chunk -c 1 -o $O/ev_ssd \
  python bench.py --config mamba2-2.7b --steps 1 --warmup 1 --no-cpu --no-e2e --layers 2 > /dev/null 2>&1
timeout 600 python scripts/dstack_trace.py > $O/ev_dstack_trace.txt 2>&1
timeout 600 python scripts/prefill_time.py --reps 5 > $O/ev_prefill_time.txt 2>&1
timeout 600 python scripts/kernel_rooflines.py --json $O/ev_rooflines.json > $O/ev_rooflines.txt 2>&1
ls -la $O/ev_*
