#!/usr/bin/env python
"""Benchmark of the tensor-parallel selective-SSM mixer path (arXiv 2602.21144) on B200.

One STEP = the whole hot path over one batch: chunked prefill of the prompt through
all layers (SSM cache populated), then token-by-token decode from the cache
(SURVEY.md §8(a) rows a1-a11), for BASELINE.json configs[1] by default:
Mamba-2.8B (64 layers, d_model 2560), batch 16, prompt 2048 + 256 decode.
Metric: batch tokens/s = B * (L_in + L_out) / (TTFT + sum of decode steps)
(SPEC.md:420-423).  TP degree = number of ranks (torchrun), so the
total work is fixed as N grows ("scaling": "strong").

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config mamba2.8b]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="mamba2.8b",
                   choices=["mamba2.8b", "falcon7b", "zamba7b", "mamba2.8b-long", "mamba2-2.7b", "tiny"],
                   help="tiny = BASELINE configs[0] (one fp32 layer, D 64, batch 2, 64 + 16): latency of the fp32 mode")
    p.add_argument("--ar2", default="int8", choices=["int8", "int8-requant", "fp16", "bf16", "fp32", "nccl"],
                   help="AR#2: int8 / fp16 / bf16 / fp32 peer-to-peer (library), or nccl = NCCL bf16 all-reduce "
                        "baseline arm")
    p.add_argument("--tp-design", default="split", choices=["split", "naive"],
                   help="split = the paper's channel splitter (2 all-reduces per block); naive = the naive sharding "
                        "baseline (2 all-gathers + 2 all-reduces per block, PAPER.md:297), TP > 1 only")
    p.add_argument("--prompt", type=int, default=0, help="override prompt length (smoke runs only)")
    p.add_argument("--decode", type=int, default=-1, help="override decode length (smoke runs only)")
    p.add_argument("--layers", type=int, default=0, help="override layer count (smoke runs only)")
    p.add_argument("--chunk", type=int, default=0, help="prefill chunk length (default: whole prompt if it fits)")

    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-pack", action="store_true", help="decode streams the row-major weights (no pre-tiled copy)")
    p.add_argument("--decode-impl", default="auto", choices=["auto", "persistent", "layer"],
                   help="persistent = one cooperative launch per token for the whole stack (TP = 1, pure Mamba "
                        "stacks); layer = the per-layer CUDA-graph decode (4 kernels per layer); auto = persistent "
                        "where supported")
    return p.parse_args()


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id):
        self.gpu_id, self.proc, self.lines = gpu_id, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu_id), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def gpu_smi_id(dev):
    import torch
    try:
        u = str(torch.cuda.get_device_properties(dev).uuid)
        return u if u.startswith("GPU-") else "GPU-" + u
    except Exception:
        return dev


# ---------------------------------------------------------------------------- oracle timing
def oracle_sample(dims, prompt, decode, batch=1):
    """Time the CPU oracle (as it stands) on a bounded sample: one layer, `batch` rows,
    `prompt` + `decode` tokens.  Returns (seconds, tokens)."""
    import numpy as np
    import synth
    from oracle import mixer_ref as M
    w = {k: v.numpy() for k, v in synth.layer_weights(dims, 0).items()}
    x, res = synth.activations(batch, prompt + decode, dims.d_model)
    x, res = x.numpy(), res.numpy()
    t0 = time.perf_counter()
    _, st = M.mixer_prefill(dims, w, x[:, :prompt], res[:, :prompt])
    for t in range(prompt, prompt + decode):
        _, st = M.mixer_decode(dims, w, x[:, t:t + 1], res[:, t:t + 1], st)
    dt = time.perf_counter() - t0
    return dt, batch * (prompt + decode)


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"), default=1)
    except Exception:
        return None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(dims, n_layers, prompt=512, decode=8, target_s=12.0):
    """Oracle on a bounded sample: one layer, batch 1, prompt + decode tokens, scaled by a power
    of two (after a calibration run) so the timed sample takes about target_s seconds of CPU."""
    dt, toks = oracle_sample(dims, prompt, decode)  # calibration
    if dt < target_s:
        f = 2 ** max(0, math.ceil(math.log2(target_s / max(dt, 1e-3))))
        prompt, decode = prompt * min(f, 256), decode * min(f, 256)
        dt, toks = oracle_sample(dims, prompt, decode)
    per_layer = toks / dt
    return {"value": per_layer / n_layers, "unit": "tokens/s", "cores": blas_threads() or len(os.sched_getaffinity(0)),
            "affinity_cores": len(os.sched_getaffinity(0)), "cpu": cpu_model(), "kind": "oracle",
            "sample": f"numpy fp64 oracle, 1 layer of {n_layers}, batch 1, prompt {prompt} + {decode} decode "
                      f"({dt:.1f} s); tokens/s extrapolated linearly to full depth (cost is linear in layers); "
                      f"GEMMs on multithreaded BLAS, per-token scan loop single-threaded"}


def run_reference(args, dims, wl, n_layers):
    """--impl reference: the oracle timed as it stands on host cores, same metric/config."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    prompt, decode = 128, 4
    for _ in range(args.warmup):
        oracle_sample(dims, 32, 1)
    secs = []
    for _ in range(args.steps):
        dt, toks = oracle_sample(dims, prompt, decode)
        secs.append(dt)
    per_layer = 1 * (prompt + decode) / statistics.mean(secs)
    value = per_layer / n_layers
    line = {"impl": "reference", "metric": "batch tokens/sec", "value": value, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * statistics.mean(secs), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {n_layers} layers, d_model {dims.d_model}, batch {wl['batch']}, "
                                   f"prompt {wl['prompt']} + {wl['decode']} decode",
                       "sample": f"per step: 1 layer, batch 1, prompt {prompt} + {decode} decode"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "kind": "oracle",
                             "cores": blas_threads() or len(os.sched_getaffinity(0)),
                             "sample": f"1 layer, batch 1, prompt {prompt} + {decode} decode per step, "
                                       f"extrapolated to {n_layers} layers"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- ranks
def launch_ranks(args):
    """`--gpus N` (N > 1) run WITHOUT torchrun: re-exec this script under torch.distributed.run with
    N ranks on this node (one process per GPU).  Fails loudly when the node has fewer GPUs."""
    import socket
    import torch
    n = torch.cuda.device_count()
    if n < args.gpus and not os.environ.get("BENCH_RANKS_SHARE_GPU"):
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but this node has {n} CUDA device(s)\n")
        sys.exit(2)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


# ---------------------------------------------------------------------------- main
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        launch_ranks(args)
    import synth
    mamba2 = args.config == "mamba2-2.7b"   # Mamba-2 (SSD) stack, SURVEY.md §8(f) NEXT-4 (not a BASELINE config)
    dims = synth.CONFIGS["mamba2.8b" if args.config in ("mamba2.8b-long", "mamba2-2.7b") else args.config]
    cdt = "fp32" if args.config == "tiny" else "bf16"   # BASELINE configs[0] is the fp32 mode
    wl = dict(synth.WORKLOADS["mamba2.8b" if mamba2 else args.config])
    n_layers = args.layers or dims.n_layers
    if args.prompt:
        wl["prompt"] = args.prompt
    if args.decode >= 0:
        wl["decode"] = args.decode
    if args.impl == "reference":
        run_reference(args, dims, wl, n_layers)
        return

    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (TP degree = number of ranks)")
    # BENCH_RANKS_SHARE_GPU=1 (test only: exercises the multi-rank launch, rendezvous and collectives on a
    # one-GPU box; the ranks' contexts are time-sliced, so its numbers are not TP measurements)
    if os.environ.get("BENCH_RANKS_SHARE_GPU"):
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if os.environ.get("BENCH_RANKS_SHARE_GPU"):  # NCCL refuses two ranks on one device
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    k = world

    from paper_2602_21144_b200 import _lib as L
    from paper_2602_21144_b200.mixer import LayerWeights, TPMixer
    from paper_2602_21144_b200.stack import MixerStack, synthetic_layer

    B, Lp, Ld = wl["batch"], wl["prompt"], wl["decode"]
    chunk = args.chunk or Lp
    while B * chunk > 65536 and chunk % 2 == 0:
        chunk //= 2
    n_chunks = math.ceil(Lp / chunk)
    flags = {"int8": L.SSM_AR2_INT8, "int8-requant": L.SSM_AR2_INT8 | L.SSM_QAR_REQUANT, "fp16": L.SSM_AR2_FP16, "bf16": L.SSM_AR2_BF16, "fp32": L.SSM_AR2_FP32,
             "nccl": L.SSM_AR2_EXTERNAL}[args.ar2]
    naive = args.tp_design == "naive" and k > 1
    if naive:
        flags |= L.SSM_TP_NAIVE

    peer_bufs, nbytes, symm, comm_kind = None, 0, None, None
    if k > 1:
        cfg = L.make_config(dims, cdt)
        nbytes = L.comm_bytes(cfg, k, B * chunk)
        try:  # peer-mapped symmetric buffers (torch symmetric memory over NVLink)
            if os.environ.get("BENCH_RANKS_SHARE_GPU"):
                raise RuntimeError("ranks share one GPU")
            import torch.distributed._symmetric_memory as symm_mem
            buf = symm_mem.empty(nbytes, dtype=torch.uint8, device=dev)
            buf.zero_()
            hdl = symm_mem.rendezvous(buf, dist.group.WORLD.group_name)
            peer_bufs = [int(p) for p in hdl.buffer_ptrs]
            symm = (buf, hdl)
            comm_kind = "symmetric_memory"
        except Exception as exc:  # the same buffers mapped by CUDA IPC handles (peer access over NVLink)
            from torch.multiprocessing.reductions import reduce_tensor
            if rank == 0:
                sys.stderr.write(f"bench.py: symmetric memory unavailable ({type(exc).__name__}: {exc}); CUDA IPC\n")
            buf = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
            torch.cuda.synchronize()
            handles = [None] * k
            dist.all_gather_object(handles, reduce_tensor(buf))
            peers = [buf if r == rank else handles[r][0](*handles[r][1]) for r in range(k)]
            peer_bufs = [int(t.data_ptr()) for t in peers]
            symm = (buf, peers)
            comm_kind = "cuda_ipc"
        dist.barrier()
    mx = TPMixer(dims, cdt, rank=rank, tp_size=k, peer_bufs=peer_bufs, buf_bytes=nbytes, device=dev)
    want_persistent = (args.decode_impl != "layer" and k == 1 and not mamba2 and args.config != "zamba7b"
                       and wl["batch"] <= 16 and cdt == "bf16")
    if args.decode_impl == "persistent" and not want_persistent:
        raise SystemExit("bench.py: --decode-impl persistent needs TP = 1, a pure Mamba stack and batch <= 16")
    layers = []
    for l in range(0 if mamba2 else n_layers):
        full = synthetic_layer(dims, l, device=dev)
        lw = LayerWeights(dims, full, k, rank, cdt, dev, naive=naive)
        if not args.no_pack and not want_persistent and cdt == "bf16":
            lw.pack(mx)  # pre-tiled copies of w_in / w_x / w_out for the decode weight streams
        layers.append(lw)
        del full
    hybrid = None
    if args.config == "zamba7b":
        # Zamba-7B: the shared attention + MLP block before its 13 hybrid layers
        from paper_2602_21144_b200.attention import hybrid_config, synthetic_shared_block
        hl = [li for li in synth.ZAMBA7B_HYBRID_LAYERS if li < n_layers]
        blk_full, lins = synthetic_shared_block(synth.ZAMBA7B_ATTN, hl, device=dev)
        hybrid = hybrid_config(synth.ZAMBA7B_ATTN, blk_full, lins, k, rank, Lp + max(Ld, 1) + 16, dev)
        del blk_full, lins
    torch.cuda.empty_cache()
    if mamba2:
        from paper_2602_21144_b200.mamba2 import Mamba2Stack, Mamba2Weights, synthetic_mamba2_layer
        m2 = synth.MAMBA2_2P7B
        m2w = []
        for l in range(n_layers):
            full = synthetic_mamba2_layer(m2, l, device=dev)
            m2w.append(Mamba2Weights(m2, full, k, rank, dev))
            del full
        torch.cuda.empty_cache()
        stack = Mamba2Stack(mx, m2, m2w, B, chunk, flags if flags != L.SSM_AR2_EXTERNAL else L.SSM_AR2_INT8)
    else:
        stack = MixerStack(mx, layers, B, chunk, flags, nccl_group=(dist.group.WORLD if k > 1 else None),
                           hybrid=hybrid)
        if want_persistent:
            try:
                stack.persistent()
            except L.SSMError as e:
                if args.decode_impl == "persistent":
                    raise
                print(f"bench.py: persistent decode unsupported here ({e}); per-layer decode", file=sys.stderr)
                for lw in layers:
                    lw.pack(mx)
    persistent = getattr(stack, "dstack", None) is not None

    # inputs: replicated on all ranks (same seed); larger than L2 (126 MB) -> no flush needed
    g = torch.Generator(device=dev).manual_seed(42)
    prompt_in = [torch.randn((B * min(chunk, Lp - c * chunk), dims.d_model), generator=g, device=dev)
                 for c in range(n_chunks)]
    dec_in = torch.randn((max(Ld, 1), B, dims.d_model), generator=g, device=dev)
    work = [p.clone() for p in prompt_in]
    res_t = torch.empty((B, dims.d_model), device=dev)
    dec_out = torch.empty((max(Ld, 1), B, dims.d_model), device=dev)
    stream = torch.cuda.current_stream()

    graph = None
    if Ld > 0:
        res_t.copy_(dec_in[0])
        # decode in_proj is timed by CUDA-event nodes inside a SECOND graph of the same step
        # (probe_graph, replayed right after the timed region): event nodes in the timed graph
        # itself would cost ~0.7 ms per step.  The probe slots stay full after this capture, so
        # the timed graph below gets no event nodes.
        probe_graph = stack.capture_decode(res_t, probes=[] if (mamba2 or persistent) else [("in_proj_decode", n_layers)])
        graph = stack.capture_decode(res_t, warmup=False)

    def prefill_part(timers=None):
        stack.reset()
        for c in range(n_chunks):
            work[c].copy_(prompt_in[c])
        if timers is not None:
            timers[0].record()
        for c in range(n_chunks):
            stack.prefill_chunk(work[c], h0=prompt_in[c])
        if timers is not None:
            timers[1].record()

    def decode_part(timers=None):
        for j in range(Ld):
            res_t.copy_(dec_in[j])
            if getattr(stack, "hybrid", None):
                stack.h0_dec.copy_(dec_in[j])
            stack.replay(graph)
            dec_out[j].copy_(res_t)
        if timers is not None:
            timers[2].record()

    def step(timers=None):
        prefill_part(timers)
        decode_part(timers)

    def barrier():
        if k > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    mx.probe("in_proj", n_layers * n_chunks * args.steps + 16)
    launches0 = mx.launches()
    timers = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(gpu_smi_id(local)) as clk:
        barrier()
        torch.cuda.synchronize()
        t_start.record()
        for i in range(args.steps):
            step(timers[i])
        t_end.record()
        torch.cuda.synchronize()
        barrier()
    pre_ms = mx.probe_read("in_proj")          # prefill in_proj launches of the timed steps
    dec_ms_launch = []
    stack_ms = []
    if Ld > 0 and persistent:
        # the persistent kernel is the whole decode step: CUDA events around single-kernel graph
        # replays on the launching stream, continuing from the timed state
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(8)]
        for j, (e0, e1) in enumerate(evs):
            res_t.copy_(dec_in[j % Ld])
            e0.record()
            stack.replay(graph)
            e1.record()
        torch.cuda.synchronize()
        stack_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    elif Ld > 0:
        for j in range(min(Ld, 8)):  # probe graph: same decode step, continuing from the timed state
            res_t.copy_(dec_in[j])
            stack.replay(probe_graph)
            dec_ms_launch += mx.probe_read("in_proj_decode")   # one per layer
    mx.probe("in_proj", 0)
    prefill_launches = mx.launches() - launches0
    total_ms = t_start.elapsed_time(t_end)
    ttft = [t[0].elapsed_time(t[1]) for t in timers]
    dec_ms = [t[1].elapsed_time(t[2]) for t in timers]
    if k > 1:
        tt = torch.tensor([total_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_step = total_ms / args.steps
    tokens = B * (Lp + Ld)
    value = tokens * args.steps / (total_ms / 1000.0)

    # e2e: same metric through the public API with host buffers (pinned H2D in, D2H out)
    e2e = None
    if not args.no_e2e:
        h_prompt = [p.cpu().pin_memory() for p in prompt_in]
        h_dec = dec_in.cpu().pin_memory()
        h_out = torch.empty_like(dec_out, device="cpu").pin_memory()
        h2d = sum(p.numel() * 4 for p in h_prompt) + h_dec.numel() * 4
        d2h = h_out.numel() * 4
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        # every step's copies are inside the timed region, pipelined on a copy stream: step i + 1's
        # prompt lands while step i decodes (after its prefill has consumed the prompt buffers), step
        # i's outputs leave and step i + 1's decode inputs land while step i + 1 prefills
        cur = torch.cuda.current_stream()
        cs = torch.cuda.Stream()
        e0.record()
        cs.wait_stream(cur)
        with torch.cuda.stream(cs):
            for c in range(n_chunks):
                prompt_in[c].copy_(h_prompt[c], non_blocking=True)
            dec_in.copy_(h_dec, non_blocking=True)
        in_ready = cs.record_event()
        dec_ready = in_ready
        for i in range(args.steps):
            cur.wait_event(in_ready)
            prefill_part()
            if i + 1 < args.steps:
                cs.wait_event(cur.record_event())
                with torch.cuda.stream(cs):
                    for c in range(n_chunks):
                        prompt_in[c].copy_(h_prompt[c], non_blocking=True)
                in_ready = cs.record_event()
            cur.wait_event(dec_ready)
            decode_part()
            cs.wait_event(cur.record_event())
            with torch.cuda.stream(cs):
                h_out.copy_(dec_out, non_blocking=True)
                if i + 1 < args.steps:
                    dec_in.copy_(h_dec, non_blocking=True)
            dec_ready = cs.record_event()
        cur.wait_event(dec_ready)
        e1.record()
        torch.cuda.synchronize()
        barrier()
        e_ms = e0.elapsed_time(e1)
        if k > 1:
            tt = torch.tensor([e_ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt.item())
        e2e = {"value": tokens * args.steps / (e_ms / 1000.0), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h}

    # roofline of the dominant kernel (largest share of the step): decode in_proj (HBM-bound weight
    # stream, swap-AB) vs prefill in_proj (tensor-core bound); both measured live with CUDA events
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    traffic = {}
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(args.config, {})
    except Exception:
        pass
    Ek, D = dims.d_inner // k, dims.d_model
    Mc = B * chunk
    roofs = {}
    if pre_ms:
        avg = statistics.mean(pre_ms)
        flops = 2 * Mc * D * 2 * Ek
        # the burst peak (cuBLAS best of 10 at full clocks) is the denominator: the in_proj runs for ~1.2 ms
        # between MUFU-bound scans, at the bench's full SM clock; the sustained (power-capped) figure beside it
        peak = peaks.get("bf16_tflops", 1614.6)
        peak_s = peaks.get("bf16_tflops_sustained", 1364.7)
        ach = flops / (avg / 1000) / 1e12
        roofs["in_proj_prefill"] = {
            "kernel": "gemm_tc_kernel (prefill in_proj, tcgen05, CTA pairs)", "bound": "tensor", "achieved": ach,
            "peak": peak, "unit": "TFLOP/s", "frac": ach / peak, "peak_sustained": peak_s,
            "frac_sustained": ach / peak_s, "traffic": traffic.get("in_proj_prefill"), "launch_ms": avg,
            "launches": len(pre_ms), "step_share_ms": sum(pre_ms) / args.steps,
            "work_per_launch": f"2*M*D*2E_k = {flops:.3e} flop (M={Mc})",
            "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst); bf16_tflops_sustained beside it"}
    if dec_ms_launch:
        avg = statistics.mean(dec_ms_launch)
        fused = stack.mx.fused_calls() > 0
        P = dims.dt_rank + 2 * dims.d_state
        es_ = 4 if cdt == "fp32" else 2
        byts = 2 * Ek * D * es_ + B * D * es_ + B * 2 * Ek * es_  # weights + x_in + xz
        if fused:  # + conv window read/write, conv taps, W_x, x_proj accumulator read/write
            byts += 2 * B * (dims.d_conv - 1) * Ek * 2 + Ek * (dims.d_conv + 1) * 4 + P * Ek * 2 + 2 * B * P * 4
        peak = peaks.get("hbm_gbs", 6535.1)
        ach = byts / (avg / 1000) / 1e9
        roofs["in_proj_decode"] = {
            "kernel": "gemm_tc_kernel (decode in_proj, swap-AB weight stream)", "bound": "hbm", "achieved": ach,
            "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": traffic.get("in_proj_decode"),
            "launch_ms": avg, "launches": len(dec_ms_launch), "step_share_ms": avg * n_layers * Ld,
            "work_per_launch": (f"W_in 2E_k*D bf16 + x_in + z + u + conv window r/w + W_x + x_proj acc = {byts:.3e} B "
                                "(in_proj with the conv step and x_proj fused into its epilogue)") if fused
                               else f"W_in 2E_k*D bf16 + x_in + xz = {byts:.3e} B",
            "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    if stack_ms:
        avg = statistics.mean(stack_ms)
        P = dims.dt_rank + 2 * dims.d_state
        E, K, N = dims.d_inner, dims.d_conv, dims.d_state
        per_layer = (2 * E * D * 2 + D * E * 2 + P * E * 2 + E * dims.dt_rank * 2     # W_in, W_out, W_x, W_dt (bf16)
                     + E * (K + 3 + N) * 4                                            # conv w/b, b_dt, D, A_log
                     + 2 * B * E * N * 4 + 2 * B * (K - 1) * E * 2)                   # h and conv window r/w
        byts = n_layers * per_layer + 2 * B * D * 4                                   # + residual in/out
        peak = peaks.get("hbm_gbs", 6535.1)
        ach = byts / (avg / 1000) / 1e9
        roofs["decode_stack"] = {
            "kernel": "decode_stack_kernel (persistent whole-stack decode, one launch per token)", "bound": "hbm",
            "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "traffic": traffic.get("decode_stack"), "launch_ms": avg, "launches": len(stack_ms),
            "step_share_ms": avg * Ld,
            "work_per_launch": (f"{n_layers} layers x (W_in + W_out + W_x + W_dt bf16 + per-channel vectors + h r/w "
                                f"+ conv window r/w = {per_layer:.4e} B) + residual = {byts:.4e} B"),
            "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    roof = max(roofs.values(), key=lambda r: r["step_share_ms"]) if roofs else None
    roof_other = [r for r in roofs.values() if r is not roof]

    cpu = None
    if rank == 0 and k == 1 and not args.no_cpu:
        cpu = cpu_baseline(dims, n_layers)

    gpu_launches = prefill_launches + args.steps * Ld * stack.graph_launches
    if rank == 0:
        line = {"metric": "batch tokens/sec", "value": value, "unit": "tokens/s", "n_gpus": k, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32" if cdt == "fp32" else "bf16", "data": "synthetic",
                "config": {"workload": f"{args.config}: {n_layers} layers"
                                       + (f" ({len(stack.hybrid)} hybrid: shared attention + MLP block first)"
                                          if getattr(stack, "hybrid", None) else "")
                                       + (" of the Mamba-2 (SSD) mixer, d_inner 5120, d_state 128, 80 heads"
                                          if mamba2 else "")
                                       + f", d_model {dims.d_model}, batch {B}, prompt {Lp} + {Ld} decode",
                           "model": args.config, "global_batch": B,
                           "seq_len": Lp + Ld, "parallelism": f"tp{k}", "ar2": args.ar2 if k > 1 else "none",
                           "tp_design": args.tp_design if k > 1 else "none", "comm": comm_kind or "none",
                           "prefill_chunk": chunk, "packed_decode_weights": not args.no_pack,
                           "decode_impl": "persistent" if persistent else "layer",
                           "l2": "inputs larger than L2 (prompt residual "
                                                         f"{B * Lp * D * 4 / 1e6:.0f} MB > 126 MB)"},
                "ttft_ms": statistics.mean(ttft), "tpot_ms": statistics.mean(dec_ms) / max(Ld, 1),
                "roofline": roof, "roofline_other": roof_other, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": gpu_launches,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if k > 1:
        torch.cuda.synchronize()
        dist.barrier()
        # release the peers' mappings (CUDA IPC: every consumer drops its handles before any owner exits)
        stack = mx = None
        symm = peer_bufs = None
        import gc
        gc.collect()
        torch.cuda.synchronize()
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
