# usage: bash run_gpu.sh TAG [tests|smoke|bench|ncu|ablate|...]...
TAG=$1; shift
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
for what in "$@"; do
case $what in
tests) timeout 900 python -m pytest tests -m gpu -q --timeout 180 -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.txt 2>&1; tail -6 gpurun_out/gpu_tests_$TAG.txt ;;
smoke) timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.txt 2>&1; tail -2 gpurun_out/smoke_$TAG.txt ;;
bench) timeout 900 python bench.py > gpurun_out/bench_$TAG.txt 2>&1; tail -1 gpurun_out/bench_$TAG.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], d['ttft_ms'], d['tpot_ms'], d['roofline']['frac'], d['clocks'])" ;;
benchq) timeout 900 python bench.py --no-cpu --no-e2e $BARGS > gpurun_out/benchq_$TAG.txt 2>&1; tail -1 gpurun_out/benchq_$TAG.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCHQ', d['value'], d['ttft_ms'], d['tpot_ms'], d['roofline']['frac'])" ;;
ncu) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --layers 2 --prompt 2048 --decode 8 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_$TAG.log 2>&1; tail -1 gpurun_out/ncu_launch_$TAG.log ;;
ablate) (for m in 0 1 8 16 24 25 31; do SSM_DEBUG_SKIP=$m timeout 120 python scripts/decode_ablation.py; done; SSM_DEBUG_SKIP_NORM=1 timeout 120 python scripts/decode_ablation.py; SSM_PDL=0 timeout 120 python scripts/decode_ablation.py) > gpurun_out/ablate_$TAG.txt 2>&1; cat gpurun_out/ablate_$TAG.txt ;;
micro) timeout 600 python scripts/gemm_micro.py > gpurun_out/micro_$TAG.txt 2>&1; cat gpurun_out/micro_$TAG.txt ;;
decexp) timeout 600 python scripts/decode_gemm_exp.py > gpurun_out/decexp_$TAG.txt 2>&1; cat gpurun_out/decexp_$TAG.txt ;;
esac
done
case " $* " in *" mk "*) 
  timeout 600 python -m pytest tests/test_gpu_stack_decode.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/mk_tests_$TAG.txt 2>&1; tail -15 gpurun_out/mk_tests_$TAG.txt
  timeout 300 python scripts/stack_decode_time.py mamba2.8b 64 > gpurun_out/mk_time_$TAG.txt 2>&1; tail -4 gpurun_out/mk_time_$TAG.txt ;;
esac
case " $* " in *" mktrace "*)
  timeout 300 python scripts/stack_trace.py mamba2.8b 16 > gpurun_out/mk_trace_$TAG.txt 2>&1; cat gpurun_out/mk_trace_$TAG.txt | tail -20 ;;
esac
case " $* " in *" mktime "*)
  timeout 300 python scripts/stack_decode_time.py mamba2.8b 64 > gpurun_out/mk_time_$TAG.txt 2>&1; tail -4 gpurun_out/mk_time_$TAG.txt ;;
esac
case " $* " in *" mkdbg "*)
  for d in 0 2; do echo "SSM_MK_DBG=$d"; SSM_MK_DBG=$d timeout 300 python scripts/stack_trace.py mamba2.8b 16 2>&1 | tail -22; done > gpurun_out/mk_dbg_$TAG.txt 2>&1; cat gpurun_out/mk_dbg_$TAG.txt ;;
esac
case " $* " in *" mkncu "*)
  for d in 0 4; do SSM_MK_DBG=$d timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:decode_mk -c 2 python scripts/stack_trace.py mamba2.8b 16 > gpurun_out/mk_ncu_${d}_$TAG.txt 2>&1; echo "DBG=$d"; grep -E "dram__|gpu__time|lts__" gpurun_out/mk_ncu_${d}_$TAG.txt | tail -5; done ;;
esac
case " $* " in *" l2probe "*)
  timeout 300 python scripts/l2_probe.py > gpurun_out/l2probe_$TAG.txt 2>&1; cat gpurun_out/l2probe_$TAG.txt | tail -8 ;;
esac
case " $* " in *" burst "*)
  timeout 300 python scripts/burst_probe.py > gpurun_out/burst_$TAG.txt 2>&1; cat gpurun_out/burst_$TAG.txt | tail -34 ;;
esac
case " $* " in *" mbar "*)
  timeout 120 python scripts/mbar_probe.py 2>&1 | tail -2 ;;
esac
case " $* " in *" mkfull "*)
  SSM_PERSISTENT_DECODE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_mk -c 1 -o gpurun_out/mk_full_$TAG python scripts/stack_trace.py mamba2.8b 16 > gpurun_out/mk_full_$TAG.log 2>&1; tail -2 gpurun_out/mk_full_$TAG.log; ls gpurun_out/ | grep mk_full ;;
esac
case " $* " in *" commitprobe "*)
  timeout 120 python scripts/commit_probe.py 2>&1 | tail -2 ;;
esac
case " $* " in *" pfab "*)
  (for v in 1 0; do SSM_L2_PREFETCH=$v timeout 120 python scripts/decode_ablation.py; SSM_L2_PREFETCH=$v SSM_DEBUG_SKIP=24 timeout 120 python scripts/decode_ablation.py; SSM_L2_PREFETCH=$v SSM_DEBUG_SKIP=8 timeout 120 python scripts/decode_ablation.py; done) > gpurun_out/pfab_$TAG.txt 2>&1; cat gpurun_out/pfab_$TAG.txt ;;
esac
case " $* " in *" kbsab "*)
  (for k in 2 3 4 6; do SSM_GEMM_KBS=$k timeout 120 python scripts/decode_ablation.py; SSM_GEMM_KBS=$k SSM_DEBUG_SKIP=24 timeout 120 python scripts/decode_ablation.py; done) > gpurun_out/kbsab_$TAG.txt 2>&1; cat gpurun_out/kbsab_$TAG.txt ;;
esac
case " $* " in *" dsfuse "*)
  (for v in 0 1; do SSM_FUSE_DSTEP=$v timeout 120 python scripts/decode_ablation.py; done) > gpurun_out/dsfuse_$TAG.txt 2>&1; cat gpurun_out/dsfuse_$TAG.txt ;;
esac
case " $* " in *" chainab "*)
  (for v in 1 0; do SSM_DECODE_CHAIN=$v timeout 120 python scripts/decode_ablation.py; done; SSM_DEBUG_SKIP=24 timeout 120 python scripts/decode_ablation.py) > gpurun_out/chainab_$TAG.txt 2>&1; cat gpurun_out/chainab_$TAG.txt ;;
esac
case " $* " in *" hlate "*)
  (for v in 0 1 0 1; do SSM_DSTEP_HLATE=$v timeout 120 python scripts/decode_ablation.py; done) > gpurun_out/hlate_$TAG.txt 2>&1; cat gpurun_out/hlate_$TAG.txt ;;
esac
case " $* " in *" l2floor "*)
  (for v in 0 1; do SSM_DSTEP_PF=$v timeout 200 python scripts/l2_floor.py; done; SSM_DEBUG_SKIP=8 timeout 200 python scripts/l2_floor.py; SSM_DEBUG_SKIP=16 timeout 200 python scripts/l2_floor.py) > gpurun_out/l2floor_$TAG.txt 2>&1; cat gpurun_out/l2floor_$TAG.txt ;;
esac
case " $* " in *" skab "*)
  (for v in 1 0 1 0; do SSM_INPROJ_SK=$v timeout 120 python scripts/decode_ablation.py; done; SSM_INPROJ_SK=1 SSM_DEBUG_SKIP=24 timeout 120 python scripts/decode_ablation.py; SSM_INPROJ_SK=1 SSM_DSTEP_PF=1 timeout 120 python scripts/decode_ablation.py) > gpurun_out/skab_$TAG.txt 2>&1; cat gpurun_out/skab_$TAG.txt ;;
esac
case " $* " in *" skprof "*)
  (for v in 0 1; do echo "SK=$v"; SSM_INPROJ_SK=$v timeout 200 python scripts/decode_profile.py; SSM_INPROJ_SK=$v SSM_PDL=0 timeout 120 python scripts/decode_ablation.py; done) > gpurun_out/skprof_$TAG.txt 2>&1; cat gpurun_out/skprof_$TAG.txt ;;
esac
case " $* " in *" skprobe "*)
  timeout 200 python scripts/sk_probe.py > gpurun_out/skprobe_$TAG.txt 2>&1; cat gpurun_out/skprobe_$TAG.txt ;;
esac
case " $* " in *" coab "*)
  (timeout 120 python scripts/decode_ablation.py; SSM_DSTEP_IPT=4 timeout 120 python scripts/decode_ablation.py;
   for r in 192 160 128; do echo "ring $r"; SSM_GEMM_RING_KB=$r timeout 120 python scripts/decode_ablation.py; SSM_DSTEP_IPT=4 SSM_GEMM_RING_KB=$r timeout 120 python scripts/decode_ablation.py; done) > gpurun_out/coab_$TAG.txt 2>&1; cat gpurun_out/coab_$TAG.txt ;;
esac
case " $* " in *" ringab "*)
  (for r in 0 192 176 160 144 112; do echo "dec ring $r"; SSM_DEC_RING_KB=$r timeout 120 python scripts/decode_ablation.py; done; echo "160+pf"; SSM_DSTEP_PF=1 timeout 120 python scripts/decode_ablation.py; echo "160 skip24"; SSM_DEBUG_SKIP=24 timeout 120 python scripts/decode_ablation.py; echo "160 skip8"; SSM_DEBUG_SKIP=8 timeout 120 python scripts/decode_ablation.py; echo "160 skip16"; SSM_DEBUG_SKIP=16 timeout 120 python scripts/decode_ablation.py) > gpurun_out/ringab_$TAG.txt 2>&1; cat gpurun_out/ringab_$TAG.txt ;;
esac
case " $* " in *" fuseab "*)
  (echo base; timeout 120 python scripts/decode_ablation.py; echo fuse_dstep; SSM_FUSE_DSTEP=1 timeout 120 python scripts/decode_ablation.py; echo chain; SSM_DECODE_CHAIN=1 timeout 120 python scripts/decode_ablation.py; echo chain+fuse; SSM_DECODE_CHAIN=1 SSM_FUSE_DSTEP=1 timeout 120 python scripts/decode_ablation.py; echo persistent; SSM_PERSISTENT_DECODE=1 timeout 120 python scripts/decode_ablation.py) > gpurun_out/fuseab_$TAG.txt 2>&1; cat gpurun_out/fuseab_$TAG.txt ;;
esac
case " $* " in *" outab "*)
  (for r in 160 128 96 64 48; do echo "out ring $r"; SSM_OUT_RING_KB=$r timeout 120 python scripts/decode_ablation.py; done; echo "out 96 ipt4"; SSM_OUT_RING_KB=96 SSM_DSTEP_IPT=4 timeout 120 python scripts/decode_ablation.py; echo "in 176 out 96"; SSM_DEC_RING_KB=176 SSM_OUT_RING_KB=96 timeout 120 python scripts/decode_ablation.py) > gpurun_out/outab_$TAG.txt 2>&1; cat gpurun_out/outab_$TAG.txt ;;
esac
case " $* " in *" scanab "*)
  (for v in 0 2 4 6 0 4; do SSM_SCAN_NP1=$v SSM_SCAN_NPOLY=$v timeout 120 python scripts/scan_micro.py; done; SSM_SCAN_VERSION=2 SSM_SCAN_NPOLY=4 timeout 120 python scripts/scan_micro.py) > gpurun_out/scanab_$TAG.txt 2>&1; cat gpurun_out/scanab_$TAG.txt ;;
esac
case " $* " in *" roof "*)
  timeout 300 python scripts/kernel_rooflines.py --json gpurun_out/rooflines_$TAG.json > gpurun_out/rooflines_$TAG.txt 2>&1; cat gpurun_out/rooflines_$TAG.txt ;;
esac
case " $* " in *" localab "*)
  (for v in 1 0 1 0; do SSM_OUT_LOCAL=$v timeout 120 python scripts/decode_ablation.py; done) > gpurun_out/localab_$TAG.txt 2>&1; cat gpurun_out/localab_$TAG.txt ;;
esac
case " $* " in *" qab "*)
  (for qk in "4 4" "2 2" "8 8" "1 1" "4 2" "8 4"; do set -- $qk; echo "Q=$1 KBS=$2"; SSM_OUT_Q=$1 SSM_OUT_KBS=$2 timeout 120 python scripts/decode_ablation.py; done; echo "off"; SSM_OUT_LOCAL=0 timeout 120 python scripts/decode_ablation.py; echo "Q4K4 gemmkbs1"; SSM_GEMM_KBS=1 timeout 120 python scripts/decode_ablation.py) > gpurun_out/qab_$TAG.txt 2>&1; cat gpurun_out/qab_$TAG.txt ;;
esac
case " $* " in *" agree "*)
  timeout 300 python -m pytest tests/test_gpu_agreement.py -q -x -p no:cacheprovider 2>&1 | tail -15
  timeout 1200 python scripts/agreement.py > gpurun_out/agreement_$TAG.jsonl 2> gpurun_out/agreement_$TAG.err; cat gpurun_out/agreement_$TAG.jsonl; tail -5 gpurun_out/agreement_$TAG.err ;;
esac
case " $* " in *" cacheab "*)
  timeout 900 python scripts/ablation_cache.py > gpurun_out/cacheab_$TAG.json 2> gpurun_out/cacheab_$TAG.err; cat gpurun_out/cacheab_$TAG.json; tail -3 gpurun_out/cacheab_$TAG.err ;;
esac
case " $* " in *" convab "*)
  (for v in 1 0; do SSM_CONV_V2=$v timeout 300 python scripts/kernel_rooflines.py --layers 2 | grep -E "conv|row"; done) > gpurun_out/convab_$TAG.txt 2>&1; cat gpurun_out/convab_$TAG.txt ;;
esac
case " $* " in *" convncu "*)
  for v in 1 0; do SSM_CONV_V2=$v timeout 600 ncu --set full --clock-control none -k regex:conv1d_silu -s 1 -c 1 -o gpurun_out/conv${v}_$TAG python bench.py --layers 2 --prompt 2048 --decode 2 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; done; ls gpurun_out/ | grep conv ;;
esac
case " $* " in *" pnab "*)
  (for v in 1 0 1 0; do SSM_PRENORM=$v timeout 120 python scripts/decode_ablation.py; done) > gpurun_out/pnab_$TAG.txt 2>&1; cat gpurun_out/pnab_$TAG.txt ;;
esac
case " $* " in *" gemmncu "*)
  A="--layers 1 --prompt 2048 --decode 0 --steps 1 --warmup 0 --no-e2e --no-cpu"
  timeout 300 python bench.py $A > gpurun_out/gemmncu_bench_$TAG.txt 2>&1; tail -c 300 gpurun_out/gemmncu_bench_$TAG.txt
  for i in 2 3; do timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s $i -c 1 -o gpurun_out/pgemm${i}_$TAG python bench.py $A > /dev/null 2>&1; done; ls gpurun_out | grep pgemm ;;
esac
case " $* " in *" zamba "*)
  timeout 900 python bench.py --config zamba7b --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/zamba_$TAG.txt 2>&1; tail -1 gpurun_out/zamba_$TAG.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ZAMBA', d['value'], d['ttft_ms'], d['tpot_ms'], d['roofline']['kernel'], d['roofline']['frac'])" ;;
esac
case " $* " in *" falcon "*)
  timeout 900 python bench.py --config falcon7b --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/falcon_$TAG.txt 2>&1; tail -1 gpurun_out/falcon_$TAG.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('FALCON', d['value'], d['ttft_ms'], d['tpot_ms'], d['roofline']['kernel'], d['roofline']['frac'])" ;;
esac
case " $* " in *" splitab "*)
  (for v in 0 1 0 1; do SSM_SCAN_SPLIT=$v timeout 120 python scripts/scan_micro.py; done; SSM_SCAN_SPLIT=1 timeout 300 python -m pytest tests -m gpu -q -x -k "scan or prefill or chunk" -p no:cacheprovider 2>&1 | tail -2) > gpurun_out/splitab_$TAG.txt 2>&1; cat gpurun_out/splitab_$TAG.txt ;;
esac
case " $* " in *" tl "*)
  timeout 300 python scripts/decode_timeline.py 8 > gpurun_out/timeline_$TAG.txt 2>&1; cat gpurun_out/timeline_$TAG.txt | tail -45 ;;
esac
case " $* " in *" fsab "*)
  (for v in 1 0 1 0; do SSM_FLAG_SYNC=$v timeout 120 python scripts/decode_ablation.py; done; SSM_PRENORM=0 timeout 120 python scripts/decode_ablation.py; timeout 120 python scripts/decode_timeline.py 4 | tail -22) > gpurun_out/fsab_$TAG.txt 2>&1; cat gpurun_out/fsab_$TAG.txt ;;
esac
case " $* " in *" xcab "*)
  (for v in 1 2 4 1 2 4; do SSM_XACC_COPIES=$v timeout 120 python scripts/decode_ablation.py | sed "s/^/copies=$v /"; done; SSM_XACC_COPIES=4 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or stack" -p no:cacheprovider 2>&1 | tail -2) > gpurun_out/xcab_$TAG.txt 2>&1; cat gpurun_out/xcab_$TAG.txt ;;
esac
case " $* " in *" splitpf "*)
  (for v in 1 0 1 0; do SSM_PREFILL_SPLIT=$v timeout 600 python bench.py --no-cpu --no-e2e --decode 8 --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('split=$v', 'ttft', round(d['ttft_ms'],1), 'tpot', round(d['tpot_ms'],3))"; done; SSM_GEMM_TRIM_RING=0 SSM_PREFILL_SPLIT=0 timeout 600 python bench.py --no-cpu --no-e2e --decode 8 --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('notrim nosplit ttft', round(d['ttft_ms'],1))") > gpurun_out/splitpf_$TAG.txt 2>&1; cat gpurun_out/splitpf_$TAG.txt ;;
esac
case " $* " in *" tpdec "*)
  cat > /tmp/tpdec.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2602_21144_b200 import _lib as L
from paper_2602_21144_b200.mixer import LayerWeights
from paper_2602_21144_b200.stack import MixerStack, synthetic_layer
from paper_2602_21144_b200.virtual import VirtualGroup
dims = synth.CONFIGS["mamba2.8b"]; B = 16; nl = 8
for k in (2, 4, 8):
    grp = VirtualGroup(dims, k, "bf16", B)
    full = [synthetic_layer(dims, l) for l in range(nl)]
    stacks = []
    for r in range(k):
        lws = [LayerWeights(dims, w, k, r, "bf16") for w in full]
        for lw in lws: lw.pack(grp.mixers[r])
        stacks.append(MixerStack(grp.mixers[r], lws, B, 1, L.SSM_AR2_INT8))
    del full
    res = [torch.randn(B, dims.d_model, device="cuda") for _ in range(k)]
    for _ in range(3):
        grp.run(lambda r, mx, s: stacks[r].decode_step(res[r], s))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        grp.run(lambda r, mx, s: stacks[r].decode_step(res[r], s))
    e1.record(); torch.cuda.synchronize()
    print(f"virtual TP={k} ({os.environ.get('SSM_FUSE_AR1','1')}): {e0.elapsed_time(e1)*1000/5/nl:.1f} us per layer-step (all k ranks on ONE GPU), fused calls {grp.mixers[0].fused_calls()}", flush=True)
    del stacks, grp; torch.cuda.empty_cache()
PY
  (for v in 1 0; do SSM_FUSE_AR1=$v timeout 300 python /tmp/tpdec.py; done) > gpurun_out/tpdec_$TAG.txt 2>&1; cat gpurun_out/tpdec_$TAG.txt | tail -8 ;;
esac
case " $* " in *" pvar "*)
  (for v in 1 0; do SSM_GEMM_PREFILL_VAR=$v timeout 300 python scripts/kernel_rooflines.py --layers 2 | grep -E "prefill" | sed "s/^/pvar=$v /"; done; for v in 1 0 1 0; do SSM_GEMM_PREFILL_VAR=$v timeout 600 python bench.py --no-cpu --no-e2e --decode 16 --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pvar=$v ttft', round(d['ttft_ms'],1))"; done) > gpurun_out/pvar_$TAG.txt 2>&1; cat gpurun_out/pvar_$TAG.txt ;;
esac
