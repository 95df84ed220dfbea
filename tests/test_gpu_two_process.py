"""TP = 2 / 4 through the REAL (non-virtual) multi-process path on one GPU: one process per rank, each with
its own CUDA context, handle (comm flags 0: PDL on, as in bench.py's torchrun path) and symmetric
buffer; the peer buffer is mapped into the other process with CUDA IPC (torch.multiprocessing
shares CUDA tensors through cudaIpcGetMemHandle / cudaIpcOpenMemHandle).  The two contexts are
time-sliced on the device, so every cross-rank barrier really waits for the other process.

Each rank runs a two-layer pre-norm stack: eager chunk-major prefill, then decode steps replayed
from a CUDA graph (MixerStack.replay realigning the epoch parity), with the int8 and the fp32
AR#2.  The replicas must be bitwise identical and match the fp64 oracle (two
all-reduces per layer; reading Q12: fixed-order reductions)."""
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synth

pytestmark = pytest.mark.gpu

DIMS = dict(d_model=256, d_inner=512, dt_rank=16, n_layers=2)
B, L_IN, L_OUT = 2, 24, 4


def _rank_main(rank, world, mode, qs, bar, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    torch.cuda.set_device(0)
    from paper_2602_21144_b200 import LayerWeights, TPMixer, _lib as L
    from paper_2602_21144_b200.stack import MixerStack, synthetic_layer
    dims = synth.MixerDims(**DIMS)
    cfg = L.make_config(dims, "bf16")
    nbytes = L.comm_bytes(cfg, world, B * L_IN)
    buf = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    for r in range(world):
        if r != rank:
            qs[r].put((rank, buf))              # CUDA IPC handle of this rank's buffer
    peers = {rank: buf}
    for _ in range(world - 1):
        r, t = qs[rank].get()
        peers[r] = t
    ptrs = [peers[r].data_ptr() for r in range(world)]
    mx = TPMixer(dims, "bf16", rank=rank, tp_size=world, peer_bufs=ptrs, buf_bytes=nbytes)
    layers = [LayerWeights(dims, synthetic_layer(dims, l), world, rank, "bf16").pack(mx) for l in range(2)]
    flags = L.SSM_AR2_INT8 if mode == "int8" else L.SSM_AR2_FP32
    stack = MixerStack(mx, layers, B, L_IN, flags)
    g = torch.Generator().manual_seed(21)
    res0 = torch.randn(B, L_IN + L_OUT, dims.d_model, generator=g, dtype=torch.float64).float()
    pre = res0[:, :L_IN].cuda().contiguous().view(B * L_IN, -1)
    res_t = torch.empty(B, dims.d_model, device="cuda")
    res_t.copy_(res0[:, L_IN].cuda())
    bar.wait()
    graph = stack.capture_decode(res_t)          # (warm-up step: collective, both ranks run it)
    stack.reset()
    stack.prefill_chunk(pre)
    outs = []
    for t in range(L_IN, L_IN + L_OUT):
        res_t.copy_(res0[:, t].cuda())
        stack.replay(graph)
        outs.append(res_t.cpu().clone())
    mx.check()
    np.save(os.path.join(out_dir, f"{mode}_pre{rank}.npy"), pre.view(B, L_IN, -1).cpu().double().numpy())
    np.save(os.path.join(out_dir, f"{mode}_dec{rank}.npy"), torch.stack(outs, 1).double().numpy())
    np.save(os.path.join(out_dir, f"{mode}_ar{rank}.npy"), np.array([mx.stats()["allreduce"], mx.launches()]))
    bar.wait()                                   # peers' mappings stay valid until everyone is done


@pytest.mark.parametrize("world,mode", [(2, "int8"), (2, "fp32"), (4, "int8")])
def test_two_process_tp_real_path_vs_oracle(tmp_path, world, mode):
    from oracle import mixer_ref as M
    from paper_2602_21144_b200.stack import synthetic_layer
    ctx = mp.get_context("spawn")
    qs = [ctx.Queue() for _ in range(world)]
    bar = ctx.Barrier(world)
    procs = [ctx.Process(target=_rank_main, args=(r, world, mode, qs, bar, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    for p in procs:
        if p.is_alive():
            p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    pre = [np.load(tmp_path / f"{mode}_pre{r}.npy") for r in range(world)]
    dec = [np.load(tmp_path / f"{mode}_dec{r}.npy") for r in range(world)]
    for r in range(1, world):                       # bitwise-identical replicas
        np.testing.assert_array_equal(pre[r], pre[0])
        np.testing.assert_array_equal(dec[r], dec[0])
    dims = synth.MixerDims(**DIMS)
    ws = []
    for l in range(2):
        full = synthetic_layer(dims, l)
        ws.append({k: (synth.bf16_round(v.cpu().double()).numpy() if k in ("w_in", "w_x", "w_dt", "w_out")
                       else v.cpu().float().double().numpy()) for k, v in full.items()})
    g = torch.Generator().manual_seed(21)
    res0 = torch.randn(B, L_IN + L_OUT, dims.d_model, generator=g, dtype=torch.float64).float().double().numpy()
    ref, _ = M.model_forward(dims, ws, res0)
    rel = lambda a, b: np.abs(a - b).max() / np.abs(b).max()
    assert rel(pre[0] - res0[:, :L_IN], ref[:, :L_IN] - res0[:, :L_IN]) < 2e-2
    assert rel(dec[0] - res0[:, L_IN:], ref[:, L_IN:] - res0[:, L_IN:]) < 2e-2
