"""world_size-2 multi-process test of the TP sharding on CPU (gloo).  What it covers: the
product's channel splitter (paper_2602_21144_b200.LayerWeights: which rows/columns each
process owns) across real processes, and the exchange structure of the method -- exactly
two all-reduces per layer.  What it does NOT cover: the library's
peer-to-peer kernels (the rank-local arithmetic here is the oracle's, the exchanges are
gloo's); those run in the -m gpu virtual-rank and two-process tests.  The replicated output
must equal the single-rank oracle, the shards must reassemble to the full weights, and the
int8 AR#2 (codes exchanged with all_gather, fixed-order sum) must give bitwise-identical
replicas within the north_star bound k max_r amax_r / 254 of the actual partials."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

DIMS = dict(d_model=64, d_inner=128, d_state=16, d_conv=4, dt_rank=4, n_layers=1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import mixer_ref as M
    from oracle import qar_ref as Q
    from paper_2602_21144_b200 import LayerWeights, channel_range

    dims = synth.MixerDims(**DIMS)
    full = synth.layer_weights(dims, 0)
    sh = LayerWeights(dims, full, world, rank, dtype="fp32", device="cpu").tensors
    sh = {k: v.double() for k, v in sh.items()}
    # (1) channel splitter: shards reassemble to the full tensors
    gathered = [None] * world
    dist.all_gather_object(gathered, {k: v.numpy() for k, v in sh.items()})
    E = dims.d_inner
    ek = E // world
    w_in_x = np.concatenate([g["w_in"][:ek] for g in gathered], 0)
    w_in_z = np.concatenate([g["w_in"][ek:] for g in gathered], 0)
    ok_split = bool(np.array_equal(np.concatenate([w_in_x, w_in_z], 0), full["w_in"].float().double().numpy())
                    and np.array_equal(np.concatenate([g["w_out"] for g in gathered], 1),
                                       full["w_out"].float().double().numpy()))
    # (2) rank-local steps + gloo all-reduces
    x, res = synth.activations(2, 10, dims.d_model, seed=3)
    x, res = x.numpy(), res.numpy()
    s = {k: v.numpy() for k, v in sh.items()}
    xl, zl = M.in_proj(x, s["w_in"])
    xc, _ = M.causal_conv1d(xl, s["conv_w"], s["conv_b"])
    u = M.silu(xc)
    part = torch.from_numpy(u @ s["w_x"].T)
    dist.all_reduce(part)                                   # AR#1
    dt_low, Bm, Cm = M.split_ssm_params(part.numpy(), dims.dt_rank, dims.d_state)
    delta = M.softplus(dt_low @ s["w_dt"].T + s["b_dt"])
    y, _ = M.scan_full(u, delta, -np.exp(s["a_log"]), Bm, Cm, s["d_skip"], np.zeros((2, ek, dims.d_state)))
    o = (y * M.silu(zl)) @ s["w_out"].T
    out = torch.from_numpy(o.copy())
    dist.all_reduce(out)                                    # AR#2 (exact)
    # (3) int8 AR#2: exchange codes + scales, fixed-order dequant-accumulate on every rank
    q, sc = Q.quantize_blocks(o.astype(np.float32).reshape(-1), 64)
    allq = [None] * world
    dist.all_gather_object(allq, (q, sc))
    acc = np.zeros(o.size)
    for qq, ss in allq:
        acc = acc + Q.dequantize_blocks(qq, ss, 64)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), res + out.numpy())
    np.save(os.path.join(out_dir, f"q{rank}.npy"), acc)
    np.save(os.path.join(out_dir, f"o{rank}.npy"), o.astype(np.float32).reshape(-1))
    with open(os.path.join(out_dir, f"ok{rank}.txt"), "w") as f:
        f.write(str(ok_split))
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_gloo_tp(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    from oracle import mixer_ref as M
    from oracle import qar_ref as Q
    dims = synth.MixerDims(**DIMS)
    w = {k: v.float().double().numpy() for k, v in synth.layer_weights(dims, 0).items()}
    x, res = synth.activations(2, 10, dims.d_model, seed=3)
    ref, _ = M.mixer_forward(dims, w, x.numpy(), res.numpy())
    r0, r1 = np.load(tmp_path / "r0.npy"), np.load(tmp_path / "r1.npy")
    np.testing.assert_array_equal(r0, r1)
    assert np.abs(r0 - ref).max() / np.abs(ref - res.numpy()).max() < 1e-12
    q0, q1 = np.load(tmp_path / "q0.npy"), np.load(tmp_path / "q1.npy")
    np.testing.assert_array_equal(q0, q1)                   # replicas bitwise identical
    parts = [np.load(tmp_path / "o0.npy"), np.load(tmp_path / "o1.npy")]
    exact = parts[0].astype(np.float64) + parts[1].astype(np.float64)
    assert np.all(np.abs(q0 - exact) <= Q.northstar_bound(parts, 64) * (1 + 1e-9))
    assert (tmp_path / "ok0.txt").read_text() == "True" and (tmp_path / "ok1.txt").read_text() == "True"
