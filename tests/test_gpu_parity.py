"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle on the same seeded
inputs (north_star tolerances: 1e-5 fp32 mode, 2e-2 bf16 I/O, normwise)."""
import numpy as np
import pytest
import torch

import synth
from oracle import mixer_ref as M
from oracle import qar_ref as Q
from oracle import tp_sim as T
from paper_2602_21144_b200 import LayerWeights, State, TPMixer, _lib as L
from gpu_helpers import (TOL, VirtualGroup, np64, oracle_state_from_gpu_layout, prep_acts, prep_weights, rel,
                               to_dev)

pytestmark = pytest.mark.gpu

MED = synth.MixerDims(d_model=256, d_inner=512, d_state=16, d_conv=4, dt_rank=16, n_layers=2)


# ------------------------------------------------------------------ GEMM
@pytest.mark.parametrize("M,N,K,swap,ks", [(300, 200, 320, 0, 1), (384, 512, 2560, 0, 1), (1000, 192, 640, 0, 1),
                                           (16, 10240 // 8, 2560, 1, 1), (16, 192, 5120, 1, 8), (32, 2560, 640, 1, 4),
                                           (5, 48, 64, 0, 1), (16, 10240, 2560, 1, 1), (32, 2560, 5120, 1, 32)])
def test_gemm_tcgen05_bf16(M, N, K, swap, ks):
    dims = synth.MixerDims(d_model=64, d_inner=128, dt_rank=4)
    mx = TPMixer(dims, "bf16")
    g = torch.Generator().manual_seed(M * 7 + N)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16)
    B = torch.randn(N, K, generator=g).to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda")
    mx.dbg_gemm(A.cuda(), B.cuda(), C, swap_ab=bool(swap), ksplit=ks)
    torch.cuda.synchronize()
    ref = A.double() @ B.double().T            # library matmul in fp64 on the same bf16 values
    assert rel(C.cpu(), ref) < 1e-5


@pytest.mark.parametrize("M,N,K,ks", [(16, 10240, 2560, 1), (16, 192, 5120, 20), (32, 2560, 5120, 7), (5, 300, 200, 1)])
def test_gemm_packed_weights(M, N, K, ks):
    """Decode GEMM streaming the pre-tiled (ssm_pack_weight) copy of W: same result as the plain layout."""
    dims = synth.MixerDims(d_model=64, d_inner=128, dt_rank=4)
    mx = TPMixer(dims, "bf16")
    g = torch.Generator().manual_seed(N + K)
    X = torch.randn(M, K, generator=g).to(torch.bfloat16)
    W = torch.randn(N, K, generator=g).to(torch.bfloat16)
    Wd = W.cuda()
    pk = mx.pack_weight(Wd)
    C = torch.empty(M, N, device="cuda")
    mx.dbg_gemm_packed(X.cuda(), Wd, pk, C, ksplit=ks)
    torch.cuda.synchronize()
    assert rel(C.cpu(), X.double() @ W.double().T) < 1e-5


@pytest.fixture
def gemm_pair():
    """Forces the CTA-pair (cta_group::2) GEMM on for every eligible call; restores the default."""
    L.call("ssm_dbg_set_gemm_pair", 1)
    yield
    L.call("ssm_dbg_set_gemm_pair", -1)


@pytest.mark.parametrize("M,N,K", [(300, 200, 320), (384, 512, 2560), (1000, 192, 640), (257, 2560, 5120),
                                   (129, 48, 64), (4096, 10240 // 4, 2560), (2048 + 77, 2560, 640)])
def test_gemm_cta_pair_bf16(gemm_pair, M, N, K):
    """The CTA-pair GEMM (two CTAs of a cluster share one 256-row UMMA tile: each loads 128 rows of
    A and half of B's rows, the leader issues cta_group::2 MMAs into both TMEMs) on ragged shapes:
    M not a multiple of 256 (the second CTA's rows partly or wholly outside A), N not a multiple of
    the tile, short and long K."""
    dims = synth.MixerDims(d_model=64, d_inner=128, dt_rank=4)
    mx = TPMixer(dims, "bf16")
    g = torch.Generator().manual_seed(M * 5 + N + K)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16)
    B = torch.randn(N, K, generator=g).to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda")
    mx.dbg_gemm(A.cuda(), B.cuda(), C)
    torch.cuda.synchronize()
    assert rel(C.cpu(), A.double() @ B.double().T) < 1e-5


@pytest.mark.parametrize("dims_name", ["med", "med_zamba"])
def test_mixer_tp1_bf16_cta_pair_gemms(gemm_pair, dims_name):
    """Every prefill projection that can run on CTA pairs does (in_proj, x_proj, dt_proj, out_proj
    with its residual add): same oracle bar as the default path."""
    dims = {"med": MED, "med_zamba": synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, n_heads=2)}[dims_name]
    gpu, ref, res, st, st_ref, _ = _run_tp1(dims, "bf16", 3, 150, 4)
    assert rel(gpu - res, ref - res) < TOL["bf16"]
    assert rel(st[1], st_ref[1]) < TOL["bf16"]


def test_gemm_simt_fp32():
    dims = synth.MixerDims(d_model=64, d_inner=128, dt_rank=4)
    mx = TPMixer(dims, "fp32")
    g = torch.Generator().manual_seed(3)
    A = torch.randn(77, 130, generator=g)
    B = torch.randn(45, 130, generator=g)
    C = torch.empty(77, 45, device="cuda")
    mx.dbg_gemm(A.cuda(), B.cuda(), C)
    torch.cuda.synchronize()
    assert rel(C.cpu(), A.double() @ B.double().T) < 1e-6


# ------------------------------------------------------------------ scan
@pytest.mark.parametrize("dtype,L_", [("fp32", 37), ("bf16", 37), ("bf16", 130)])
def test_scan_kernel_vs_oracle(dtype, L_):
    dims = synth.MixerDims(d_model=128, d_inner=384, d_state=16, dt_rank=8)
    mx = TPMixer(dims, dtype)
    B, E, N = 2, 384, 16
    g = torch.Generator().manual_seed(5)
    rnd = lambda *s: torch.randn(*s, generator=g, dtype=torch.float64)
    u = rnd(B, L_, E)
    delta = torch.exp(torch.rand(B, L_, E, generator=g, dtype=torch.float64) * 4.6 - 6.9)   # 1e-3 .. 1e-1
    z = rnd(B, L_, E)
    BC = rnd(B, L_, 2 * N)
    w = prep_weights(dims, 0, dtype)
    a_log, d_skip = w["a_log"], w["d_skip"]
    h0 = rnd(B, E, N) * 0.5
    if dtype == "bf16":
        u, delta, z = synth.bf16_round(u), synth.bf16_round(delta), synth.bf16_round(z)
    BC = BC.to(torch.float32).double()
    h0 = h0.to(torch.float32).double()
    h = h0.to(torch.float32).cuda()
    gout = torch.empty(B * L_, E, dtype=torch.bfloat16 if dtype == "bf16" else torch.float32, device="cuda")
    mx.dbg_scan(to_dev(u, dtype), to_dev(delta, dtype), to_dev(z, dtype), E, BC.float().cuda(),
                a_log.float().cuda(), d_skip.float().cuda(), h, gout, B, L_)
    torch.cuda.synchronize()
    A = -np.exp(a_log.numpy())
    y, hL = M.scan_full(u.numpy(), delta.numpy(), A, BC[..., :N].numpy(), BC[..., N:].numpy(), d_skip.numpy(),
                        h0.numpy())
    gref = y * M.silu(z.numpy())
    assert rel(gout.float().cpu().view(B, L_, E), gref) < TOL[dtype]
    assert rel(h.cpu(), hL) < TOL[dtype]
    # the state is fp32 and the inputs are exactly the oracle's, so only the exp2 (MUFU ex2 or the
    # FMA-pipe polynomial, both ~2.4e-7 relative) and fp32 rounding separate h from the oracle
    assert rel(h.cpu(), hL) < 1e-4


# ------------------------------------------------------------------ full mixer, TP=1
def _run_tp1(dims, dtype, B, L_in, L_out, chunks=None, layer=0, pack=False, dec_flags=L.SSM_AR2_INT8):
    w = prep_weights(dims, layer, dtype)
    x, res = prep_acts(B, L_in + L_out, dims, dtype, seed=11 + layer)
    mx = TPMixer(dims, dtype)
    lw = LayerWeights(dims, w, dtype=dtype)
    if pack:
        lw.pack(mx)
    st = State(mx, B)
    outs = []
    chunks = chunks or [L_in]
    t0 = 0
    for c in chunks:
        xi = to_dev(x[:, t0:t0 + c], dtype).view(B * c, -1)
        r = res[:, t0:t0 + c].float().cuda().contiguous().view(B * c, -1)
        mx.prefill(lw, st, xi, r)
        outs.append(r.view(B, c, -1))
        t0 += c
    for t in range(L_in, L_in + L_out):
        xi = to_dev(x[:, t:t + 1], dtype).view(B, -1)
        r = res[:, t:t + 1].float().cuda().contiguous().view(B, -1)
        mx.decode(lw, st, xi, r, dec_flags)
        outs.append(r.view(B, 1, -1))
    torch.cuda.synchronize()
    gpu = torch.cat([o.cpu() for o in outs], 1).double().numpy()
    ref, st_ref = M.mixer_forward(dims, np64(w), x.numpy(), res.numpy())
    conv, h = oracle_state_from_gpu_layout(st.conv, st.h)
    return gpu, ref, res.numpy(), (conv, h), st_ref, mx


def test_mixer_tp1_fp32_tiny_prefill_decode():
    dims = synth.CONFIGS["tiny"]
    wl = synth.WORKLOADS["tiny"]
    gpu, ref, res, st, st_ref, _ = _run_tp1(dims, "fp32", wl["batch"], wl["prompt"], wl["decode"])
    assert rel(gpu - res, ref - res) < TOL["fp32"]
    assert rel(st[1], st_ref[1]) < TOL["fp32"]
    assert rel(st[0], st_ref[0]) < TOL["fp32"]


@pytest.mark.parametrize("dims_name,pack", [("med", False), ("med_falcon", False), ("med_zamba", False),
                                            ("med", True), ("med_zamba", True), ("med_r32", False),
                                            ("med_zamba_r32", False), ("med_falcon_r32", False)])
def test_mixer_tp1_bf16_prefill_decode(dims_name, pack):
    """TP = 1 bf16 prefill + decode vs the oracle.  dt_rank 32 (P a multiple of 32): the x_proj epilogue
    writes dt_low (bf16) and B || C (fp32) itself (EPI_SPLIT_DBC, per head for Zamba; Falcon keeps the
    unpack pass for its dt/B/C RMSNorm)."""
    dims = {"med": MED,
            "med_falcon": synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, bcdt_rmsnorm=True),
            "med_zamba": synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, n_heads=2),
            "med_r32": synth.MixerDims(d_model=256, d_inner=512, dt_rank=32),
            "med_zamba_r32": synth.MixerDims(d_model=256, d_inner=512, dt_rank=32, n_heads=2),
            "med_falcon_r32": synth.MixerDims(d_model=256, d_inner=512, dt_rank=32, bcdt_rmsnorm=True)}[dims_name]
    gpu, ref, res, st, st_ref, mx = _run_tp1(dims, "bf16", 3, 150, 6, pack=pack)
    assert rel(gpu - res, ref - res) < TOL["bf16"]
    assert rel(st[1], st_ref[1]) < TOL["bf16"]
    assert rel(st[0], st_ref[0]) < TOL["bf16"]
    assert mx.stats()["allreduce"] == 0         # TP=1: no all-reduce (reading Q13)


@pytest.mark.parametrize("B,dims_name", [(1, "med"), (16, "med"), (17, "med"), (32, "med"), (5, "med_zamba"),
                                         (4, "med_falcon"), (16, "med_zamba_wide")])
def test_fused_decode_inproj_matches_unfused_and_oracle(B, dims_name):
    """Decode in_proj with the conv step and x_proj fused into its epilogue (tokens split over
    the two epilogue halves, x_proj partials accumulated into the state's zeroed buffer and
    re-zeroed by out_proj) against the unfused kernel chain (SSM_DECODE_UNFUSED) and the oracle,
    over several steps."""
    dims = {"med": MED,
            "med_falcon": synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, bcdt_rmsnorm=True),
            "med_zamba": synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, n_heads=2),
            # P = dt_rank + 2 d_state = 272 > 256 (Zamba-7B: 264): the fused path's widest x_proj
            "med_zamba_wide": synth.MixerDims(d_model=256, d_inner=512, dt_rank=240, n_heads=2)}[dims_name]
    res = {}
    for fuse in (True, False):
        flags = L.SSM_AR2_INT8 | (0 if fuse else L.SSM_DECODE_UNFUSED)
        gpu, ref, r0, st, st_ref, mx = _run_tp1(dims, "bf16", B, 40, 5, pack=True, dec_flags=flags)
        assert rel(gpu - r0, ref - r0) < TOL["bf16"], fuse
        assert rel(st[1], st_ref[1]) < TOL["bf16"], fuse
        assert rel(st[0], st_ref[0]) < TOL["bf16"], fuse
        assert mx.fused_calls() == (5 if fuse else 0)
        res[fuse] = (gpu, st)
    # same arithmetic up to the x_proj summation order: the paths agree far inside the tolerance
    assert rel(res[True][0] - r0, res[False][0] - r0) < 5e-3
    np.testing.assert_array_equal(res[True][1][0], res[False][1][0])   # conv window: raw x values


def test_mixer_chunked_prefill_matches_oracle_and_is_chunk_invariant():
    dims = MED
    g1, ref, res, st1, _, _ = _run_tp1(dims, "bf16", 2, 100, 0)
    g2, _, _, st2, _, _ = _run_tp1(dims, "bf16", 2, 100, 0, chunks=[1, 30, 3, 66])
    assert rel(g2 - res, ref - res) < TOL["bf16"]
    assert rel(g2 - res, g1 - res) < TOL["bf16"]
    assert rel(st2[1], st1[1]) < TOL["bf16"]
    np.testing.assert_array_equal(st2[0], st1[0])     # conv window holds raw x values


def test_mixer_fp32_edge_cases():
    dims = synth.CONFIGS["tiny"]
    # L=1 prefill, L < K-1 chunks mixing old state and new input, batch 1
    g, ref, res, st, st_ref, _ = _run_tp1(dims, "fp32", 1, 5, 3, chunks=[1, 2, 2])
    assert rel(g - res, ref - res) < TOL["fp32"]
    assert rel(st[1], st_ref[1]) < TOL["fp32"]


def test_api_errors_on_gpu():
    dims = MED
    mx = TPMixer(dims, "bf16")
    other = TPMixer(dims, "bf16")
    st = State(other, 2)
    w = LayerWeights(dims, prep_weights(dims, 0, "bf16"))
    x = torch.zeros(2 * 4, dims.d_model, dtype=torch.bfloat16, device="cuda")
    r = torch.zeros(2 * 4, dims.d_model, device="cuda")
    with pytest.raises(L.SSMError) as e:
        mx.prefill(w, st, x, r)
    assert e.value.name == "SSM_ERR_CACHE"
    st2 = State(mx, 2)
    with pytest.raises(L.SSMError) as e:
        mx.prefill(w, st2, x, r, workspace=torch.empty(256, dtype=torch.uint8, device="cuda"))
    assert e.value.name == "SSM_ERR_ARG"


# ------------------------------------------------------------------ virtual TP (single GPU, k streams)
def _tp_virtual(dims, dtype, k, B, L_in, L_out, flags, qar_block=128, naive=False):
    """All device inputs and workspaces are created BEFORE the ranks' work is enqueued:
    a pageable H2D copy or a cudaMalloc inside the enqueue loop can serialise against a
    spinning peer barrier of another virtual rank on the same device."""
    w = prep_weights(dims, 0, dtype)
    x, res = prep_acts(B, L_in + L_out, dims, dtype, seed=17)
    grp = VirtualGroup(dims, k, dtype, B * max(L_in, 1), qar_block)
    lws = [LayerWeights(dims, w, k, r, dtype, naive=naive) for r in range(k)]
    sts = [State(grp.mixers[r], B) for r in range(k)]
    ws_p = [grp.mixers[r].workspace(B, L_in, flags) for r in range(k)]
    ws_d = [grp.mixers[r].workspace(B, 1, flags) for r in range(k)]
    xp = [to_dev(x[:, :L_in], dtype).view(B * L_in, -1) for _ in range(k)]
    rp = [res[:, :L_in].float().cuda().contiguous().view(B * L_in, -1) for _ in range(k)]
    xd = [[to_dev(x[:, t:t + 1], dtype).view(B, -1) for t in range(L_in, L_in + L_out)] for _ in range(k)]
    rd = [[res[:, t:t + 1].float().cuda().contiguous().view(B, -1) for t in range(L_in, L_in + L_out)]
          for _ in range(k)]
    torch.cuda.synchronize()
    grp.run(lambda r, mx, s: mx.prefill(lws[r], sts[r], xp[r], rp[r], flags=flags, workspace=ws_p[r], stream=s))
    for j in range(L_out):
        grp.run(lambda r, mx, s, j=j: mx.decode(lws[r], sts[r], xd[r][j], rd[r][j], flags=flags, workspace=ws_d[r],
                                                stream=s))
    outs = [torch.cat([rp[r].view(B, L_in, -1)] + [o.view(B, 1, -1) for o in rd[r]], 1).cpu() for r in range(k)]
    return outs, w, x, res, grp, sts


@pytest.mark.parametrize("k,mode", [(2, "int8"), (4, "int8"), (2, "fp32"), (4, "fp32")])
def test_virtual_tp_mixer_vs_oracle(k, mode):
    dims = MED
    flags = L.SSM_AR2_INT8 if mode == "int8" else L.SSM_AR2_FP32
    outs, w, x, res, grp, sts = _tp_virtual(dims, "bf16", k, 2, 40, 4, flags)
    # replicas bitwise identical on every rank (fixed-order reductions, reading Q12 / H7)
    for r in range(1, k):
        assert torch.equal(outs[r], outs[0])
    ref, st_ref = M.mixer_forward(dims, np64(w), x.numpy(), res.numpy())
    resn = res.numpy()
    assert rel(outs[0].double().numpy() - resn, ref - resn) < TOL["bf16"]
    # per-rank cache shard == oracle channel slice
    h = np.concatenate([sts[r].h.cpu().double().numpy() for r in range(k)], 1)
    assert rel(h, st_ref[1]) < TOL["bf16"]
    # exactly two all-reduces per layer call
    assert grp.mixers[0].stats()["allreduce"] == 2 * (1 + 4)


def test_virtual_tp_zamba_heads_k2_one_allreduce():
    dims = synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, n_heads=2)
    outs, w, x, res, grp, _ = _tp_virtual(dims, "bf16", 2, 2, 24, 2, L.SSM_AR2_FP32)
    ref, _ = M.mixer_forward(dims, np64(w), x.numpy(), res.numpy())
    resn = res.numpy()
    assert rel(outs[0].double().numpy() - resn, ref - resn) < TOL["bf16"]
    assert grp.mixers[0].stats()["allreduce"] == 1 * 3       # head-aligned shards: no AR#1 (Q17)


@pytest.mark.parametrize("k", [2, 4, 8])
def test_virtual_qallreduce_codes_bitexact_and_bound(k):
    dims = MED
    n = 6 * dims.d_model
    parts = synth.partials(k, n, seed=100 + k)
    grp = VirtualGroup(dims, k, "bf16", 64)
    outs = [torch.empty(n, device="cuda") for _ in range(k)]
    dev_parts = [parts[r].cuda() for r in range(k)]
    grp.run(lambda r, mx, s: mx.qallreduce(dev_parts[r], outs[r], stream=s))
    res_ref, codes, scales = Q.qallreduce(list(parts.numpy()), 128)
    # epoch 1 -> half 1 of each rank's symmetric buffer: codes at 0, scales at align256(n)
    half = ((grp.bufs[0].numel() - 256) // 2) & ~255
    for r in range(k):
        base = 256 + half
        q = grp.bufs[r][base:base + n].cpu().view(torch.int8).numpy()
        soff = base + ((n + 255) // 256) * 256
        s = grp.bufs[r][soff:soff + 4 * (n // 128)].cpu().view(torch.float32).numpy()
        np.testing.assert_array_equal(q, codes[r])
        np.testing.assert_array_equal(s, scales[r])
    for r in range(1, k):
        assert torch.equal(outs[r], outs[0])
    got = outs[0].cpu().double().numpy()
    assert np.abs(got - res_ref).max() <= 1e-6 * np.abs(res_ref).max()
    exact = parts.double().sum(0).numpy()
    assert np.all(np.abs(got - exact) <= Q.northstar_bound(list(parts.numpy()), 128) * (1 + 1e-5) + 1e-7)


@pytest.mark.parametrize("k", [2, 4, 8])
def test_virtual_fp16_allreduce_bitexact(k):
    """The paper's FP32 -> FP16 wire: wire bytes and the fp32 rank-order sum
    equal the oracle bit for bit; the error stays within the fp16 bound."""
    dims = MED
    n = 6 * dims.d_model
    parts = synth.partials(k, n, seed=200 + k)
    grp = VirtualGroup(dims, k, "bf16", 64)
    outs = [torch.empty(n, device="cuda") for _ in range(k)]
    dev_parts = [parts[r].cuda() for r in range(k)]
    grp.run(lambda r, mx, s: mx.qallreduce(dev_parts[r], outs[r], stream=s, fp16=True))
    ref, wire = Q.fp16_allreduce(list(parts.numpy()))
    half = ((grp.bufs[0].numel() - 256) // 2) & ~255
    for r in range(k):
        base = 256 + half  # epoch 1 -> half 1
        h = grp.bufs[r][base:base + 2 * n].cpu().view(torch.float16).numpy()
        np.testing.assert_array_equal(h.view(np.uint16), wire[r].view(np.uint16))
    for r in range(k):
        np.testing.assert_array_equal(outs[r].cpu().numpy(), ref)
    exact = parts.double().sum(0).numpy()
    assert np.all(np.abs(outs[0].cpu().double().numpy() - exact) <= Q.fp16_error_bound(list(parts.numpy())))


@pytest.mark.parametrize("k", [2, 4, 8])
def test_virtual_bf16_allreduce_bitexact(k):
    """The custom bf16 wire: wire bytes and the fp32 rank-order sum equal the oracle bit for bit;
    the error stays within the bf16 bound."""
    dims = MED
    n = 6 * dims.d_model
    parts = synth.partials(k, n, seed=250 + k)
    grp = VirtualGroup(dims, k, "bf16", 64)
    outs = [torch.empty(n, device="cuda") for _ in range(k)]
    dev_parts = [parts[r].cuda() for r in range(k)]
    grp.run(lambda r, mx, s: mx.qallreduce(dev_parts[r], outs[r], stream=s, bf16=True))
    ref, wire = Q.bf16_allreduce(list(parts.numpy()))
    half = ((grp.bufs[0].numel() - 256) // 2) & ~255
    for r in range(k):
        base = 256 + half  # epoch 1 -> half 1
        h = grp.bufs[r][base:base + 2 * n].cpu().view(torch.int16).numpy().view(np.uint16)
        np.testing.assert_array_equal(h, (wire[r].view(np.uint32) >> 16).astype(np.uint16))
    for r in range(k):
        np.testing.assert_array_equal(outs[r].cpu().numpy(), ref)
    exact = parts.double().sum(0).numpy()
    assert np.all(np.abs(outs[0].cpu().double().numpy() - exact) <= Q.bf16_error_bound(list(parts.numpy())))


@pytest.mark.parametrize("k,arm", [(2, "twoshot"), (4, "twoshot"), (8, "twoshot"), (4, "fp16"), (4, "bf16")])
def test_virtual_allreduce_accumulate_bitexact(k, arm):
    """SSM_QAR_ACCUMULATE (the mixer's mode: the result is added to the fp32 residual): out =
    fl32(residual + result), the result rounded as the oracle rounds it (fl32(s * Q) for the
    two-shot all-gather: no fma contraction with the residual add)."""
    dims = MED
    n = 6 * dims.d_model
    parts = synth.partials(k, n, seed=400 + k)
    g = torch.Generator().manual_seed(k)
    res0 = (torch.randn(n, generator=g) * 3).float()
    grp = VirtualGroup(dims, k, "bf16", 64)
    outs = [res0.clone().cuda() for _ in range(k)]
    dev_parts = [parts[r].cuda() for r in range(k)]
    kw = {"twoshot": dict(twoshot=True), "fp16": dict(fp16=True), "bf16": dict(bf16=True)}[arm]
    grp.run(lambda r, mx, s: mx.qallreduce(dev_parts[r], outs[r], accumulate=True, stream=s, **kw))
    if arm == "twoshot":
        ref, _, _ = Q.qallreduce_twoshot(list(parts.numpy()), 128)
    elif arm == "fp16":
        ref, _ = Q.fp16_allreduce(list(parts.numpy()))
    else:
        ref, _ = Q.bf16_allreduce(list(parts.numpy()))
    want = (res0.numpy() + ref).astype(np.float32)
    for r in range(k):
        np.testing.assert_array_equal(outs[r].cpu().numpy(), want)


@pytest.mark.parametrize("k", [2, 4, 8])
def test_virtual_qallreduce_twoshot_bitexact(k):
    """Two-shot shared-scale int8 schedule (reading Q6): codes, scales and the result equal the
    oracle bit for bit on every rank; error within k max|x| / 254."""
    dims = MED
    n = 6 * dims.d_model
    parts = synth.partials(k, n, seed=300 + k)
    grp = VirtualGroup(dims, k, "bf16", 64)
    outs = [torch.empty(n, device="cuda") for _ in range(k)]
    dev_parts = [parts[r].cuda() for r in range(k)]
    grp.run(lambda r, mx, s: mx.qallreduce(dev_parts[r], outs[r], stream=s, twoshot=True))
    ref, codes, scales = Q.qallreduce_twoshot(list(parts.numpy()), 128)
    half = ((grp.bufs[0].numel() - 256) // 2) & ~255
    a256 = lambda b: (b + 255) // 256 * 256
    nb = n // 128
    for r in range(k):
        base = 256 + half  # epoch 1 -> half 1: amax | scale | codes | sums
        sc = grp.bufs[r][base + a256(4 * nb):base + a256(4 * nb) + 4 * nb].cpu().view(torch.float32).numpy()
        q = grp.bufs[r][base + 2 * a256(4 * nb):base + 2 * a256(4 * nb) + n].cpu().view(torch.int8).numpy()
        np.testing.assert_array_equal(sc, scales)
        np.testing.assert_array_equal(q, codes[r])
        np.testing.assert_array_equal(outs[r].cpu().numpy(), ref)
    exact = parts.double().sum(0).numpy()
    assert np.all(np.abs(outs[0].cpu().double().numpy() - exact) <= Q.northstar_bound(list(parts.numpy()), 128) * (1 + 1e-5))


@pytest.mark.parametrize("k,sched", [(4, L.SSM_QAR_TWOSHOT), (4, L.SSM_QAR_ONESHOT), (8, 0)])
def test_virtual_tp_mixer_int8_schedules_vs_oracle(k, sched):
    dims = MED
    outs, w, x, res, grp, sts = _tp_virtual(dims, "bf16", k, 2, 40, 4, L.SSM_AR2_INT8 | sched)
    for r in range(1, k):
        assert torch.equal(outs[r], outs[0])
    ref, _ = M.mixer_forward(dims, np64(w), x.numpy(), res.numpy())
    resn = res.numpy()
    assert rel(outs[0].double().numpy() - resn, ref - resn) < TOL["bf16"]


@pytest.mark.parametrize("k", [2, 4])
@pytest.mark.parametrize("wire", ["fp16", "bf16"])
def test_virtual_tp_mixer_w16_ar2_vs_oracle(k, wire):
    dims = MED
    flags = L.SSM_AR2_FP16 if wire == "fp16" else L.SSM_AR2_BF16
    outs, w, x, res, grp, sts = _tp_virtual(dims, "bf16", k, 2, 40, 4, flags)
    for r in range(1, k):
        assert torch.equal(outs[r], outs[0])
    ref, _ = M.mixer_forward(dims, np64(w), x.numpy(), res.numpy())
    resn = res.numpy()
    assert rel(outs[0].double().numpy() - resn, ref - resn) < TOL["bf16"]
    assert grp.mixers[0].stats()["allreduce"] == 2 * (1 + 4)


def test_rmsnorm_kernel():
    dims = MED
    mx = TPMixer(dims, "fp32")
    g = torch.Generator().manual_seed(9)
    x = torch.randn(37, dims.d_model, generator=g, dtype=torch.float64)
    w = torch.rand(dims.d_model, generator=g, dtype=torch.float64)
    y = torch.empty(37, dims.d_model, device="cuda")
    mx.rmsnorm(x.float().cuda(), y, w.float().cuda(), eps=1e-5)
    torch.cuda.synchronize()
    assert rel(y.cpu(), M.rmsnorm(x.numpy(), w.numpy(), 1e-5)) < 1e-6


@pytest.mark.parametrize("k,mode,L_in", [(2, "int8", 12), (4, "fp32", 12), (4, "int8", 40), (8, "int8", 12)])
def test_virtual_tp_stack_prefill_then_graph_decode(k, mode, L_in):
    """Two-layer pre-norm stack on k virtual ranks: eager chunked prefill, then decode steps
    replayed from per-rank CUDA graphs (device-side AR epochs, alternating buffer halves).  With the
    int8 AR#2 the prefill runs ssm_mixer_prefill_normed at TP > 1: the one-shot reduce (k = 2, 8 at
    24 tokens) or the two-shot all-gather (k = 4 at 80 tokens) writes the next layer's bf16 input and
    row sums of squares -- no normalisation pass."""
    from paper_2602_21144_b200.stack import MixerStack
    dims = synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, n_layers=2)
    B, L_out = 2, 3
    flags = L.SSM_AR2_INT8 if mode == "int8" else L.SSM_AR2_FP32
    ws = [prep_weights(dims, l, "bf16") for l in range(2)]
    g = torch.Generator().manual_seed(5)
    res0 = torch.randn(B, L_in + L_out, dims.d_model, generator=g, dtype=torch.float64).float().double()
    grp = VirtualGroup(dims, k, "bf16", B * L_in)
    stacks = [MixerStack(grp.mixers[r], [LayerWeights(dims, w, k, r, "bf16") for w in ws], B, L_in, flags)
              for r in range(k)]
    assert stacks[0].prefill_normed == (mode == "int8")
    pre = [res0[:, :L_in].float().cuda().contiguous().view(B * L_in, -1) for _ in range(k)]
    rt = [torch.empty(B, dims.d_model, device="cuda") for _ in range(k)]
    torch.cuda.synchronize()
    grp.run(lambda r, mx, s: stacks[r].prefill_chunk(pre[r], s))
    # graphs: capture each rank's decode step (capture does not execute, so no cross-rank wait)
    graphs = []
    for r in range(k):
        with torch.cuda.stream(grp.streams[r]):
            graphs.append(stacks[r].capture_decode(rt[r], warmup=False))
    outs = [[] for _ in range(k)]
    for t in range(L_in, L_in + L_out):
        for r in range(k):
            rt[r].copy_(res0[:, t].float().cuda())
        torch.cuda.synchronize()
        if t == L_in + 1:  # an eager collective between replays flips the epoch parity ...
            grp.run(lambda r, mx, s: mx.barrier(s))
            assert all(mx.epoch() & 1 != stacks[0]._graph_parity for mx in grp.mixers)
        grp.run(lambda r, mx, s: stacks[r].replay(graphs[r], s))  # ... which replay() realigns
        assert all(mx.epoch() & 1 == stacks[0]._graph_parity for mx in grp.mixers)
        for r in range(k):
            outs[r].append(rt[r].cpu().clone())
    for r in range(1, k):
        assert torch.equal(pre[r].cpu(), pre[0].cpu())
        for j in range(L_out):
            assert torch.equal(outs[r][j], outs[0][j])
    ref, _ = M.model_forward(dims, [np64(w) for w in ws], res0.numpy())
    got_pre = pre[0].view(B, L_in, -1).cpu().double().numpy()
    got_dec = torch.stack(outs[0], 1).double().numpy()
    r0 = res0.numpy()
    assert rel(got_pre - r0[:, :L_in], ref[:, :L_in] - r0[:, :L_in]) < TOL["bf16"]
    assert rel(got_dec - r0[:, L_in:], ref[:, L_in:] - r0[:, L_in:]) < TOL["bf16"]


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_degenerate_softplus_linear_branch_and_full_decay(dtype, monkeypatch):
    """Degenerate regimes of the method (reading Q2): dt_proj bias so large that
    softplus takes its linear branch (v > 20) and decays exp(dt A) underflow to 0 (h forgets
    everything each step), plus a zero-bias half where softplus(v) ~ ln 2 -- prefill and decode
    against the oracle."""
    dims = synth.CONFIGS["tiny"] if dtype == "fp32" else MED
    B, L_in, L_out = 2, 24, 3
    w = prep_weights(dims, 0, dtype)
    E = dims.d_inner
    w["b_dt"] = w["b_dt"].clone()
    w["b_dt"][: E // 2] = 25.0                 # softplus linear branch, decay exp(-25 e^{A_log}) -> 0
    w["b_dt"][E // 2:] = 0.0
    x, res = prep_acts(B, L_in + L_out, dims, dtype, seed=5)
    mx = TPMixer(dims, dtype)
    lw = LayerWeights(dims, w, dtype=dtype)
    st = State(mx, B)
    xi = to_dev(x[:, :L_in], dtype).view(B * L_in, -1)
    r = res[:, :L_in].float().cuda().contiguous().view(B * L_in, -1)
    mx.prefill(lw, st, xi, r)
    outs = [r.view(B, L_in, -1)]
    for t in range(L_in, L_in + L_out):
        rt = res[:, t].float().cuda().contiguous()
        mx.decode(lw, st, to_dev(x[:, t], dtype), rt)
        outs.append(rt.view(B, 1, -1))
    torch.cuda.synchronize()
    gpu = torch.cat([o.cpu() for o in outs], 1).double().numpy()
    ref, st_ref = M.mixer_forward(dims, np64(w), x.numpy(), res.numpy())
    resn = res.numpy()
    assert rel(gpu - resn, ref - resn) < TOL[dtype]
    _, h = oracle_state_from_gpu_layout(st.conv, st.h)
    assert rel(h, st_ref[1]) < TOL[dtype]


def test_long_prompt_64k_single_chunk():
    """The cfg5 prompt length (65536 tokens, the longest sequence the bench runs) as ONE prefill
    call of 2 x 65536 = 131072 rows, then two decode steps, against the oracle (narrow channels so
    the fp64 oracle stays quick; the scan carries its state across all 65536 steps)."""
    import test_gpu_fullsize as F
    F._run(MED, 2, 65536, 2, rows=(0, 1))


def test_empty_calls_are_noops_and_state_untouched():
    """Empty inputs: prefill with seqlen 0 and qallreduce with n = 0 return OK without touching the
    residual or the cache (SPEC.md:162, 172 shapes; reading Q19: chunking, including empty
    chunks, must not change the result)."""
    dims = MED
    mx = TPMixer(dims, "bf16")
    w = LayerWeights(dims, prep_weights(dims, 0, "bf16"))
    st = State(mx, 2)
    x, res = prep_acts(2, 6, dims, "bf16", seed=3)
    xi = to_dev(x, "bf16").view(12, -1)
    r = res.float().cuda().contiguous().view(12, -1)
    mx.prefill(w, st, xi, r)
    torch.cuda.synchronize()
    h0, c0, r0 = st.h.clone(), st.conv.clone(), r.clone()
    e = torch.empty(0, dims.d_model, device="cuda")
    L.call("ssm_mixer_prefill", mx.handle, __import__("ctypes").byref(w.struct), st.handle, xi.data_ptr(),
           r.data_ptr(), 2, 0, L.SSM_AR2_INT8, mx.workspace(2, 1).data_ptr(), mx.workspace_bytes(2, 1), None)
    zbuf = torch.full((128,), 7.0, device="cuda")
    mx.qallreduce(zbuf[:0], zbuf[:0])            # n = 0 (valid pointers): no work
    torch.cuda.synchronize()
    assert torch.equal(st.h, h0) and torch.equal(st.conv, c0) and torch.equal(r, r0)
    assert torch.all(zbuf == 7.0)
    del e


@pytest.mark.parametrize("k,qblk,pair", [(2, 128, 0), (4, 128, 0), (2, 64, 0), (2, 128, 1), (4, 64, 1)])
def test_prefill_out_proj_quant_epilogue_bitexact(k, qblk, pair):
    """a8 fused: at prefill with the one-shot int8 schedule the out_proj epilogue quantises its TMEM
    accumulator straight into the symmetric buffer.  Its codes and scales must equal qar_ref's
    quantisation of the rank's fp32 partial (taken from the same prefill run with SSM_AR2_EXTERNAL,
    which writes that partial instead) bit for bit (reading Q6-Q8).  pair = 1: every eligible GEMM on
    CTA pairs (the quantising drain then runs in both CTAs of a pair)."""
    L.call("ssm_dbg_set_gemm_pair", pair if pair else -1)
    try:
        _quant_epilogue_bitexact(k, qblk, 2, 150 if pair else 40)
    finally:
        L.call("ssm_dbg_set_gemm_pair", -1)


def _quant_epilogue_bitexact(k, qblk, B, Lp):
    dims = MED
    w = prep_weights(dims, 0, "bf16")
    x, res = prep_acts(B, Lp, dims, "bf16", seed=23)
    n = B * Lp * dims.d_model
    parts, codes, scales = [], [], []
    for mode in ("external", "int8"):
        grp = VirtualGroup(dims, k, "bf16", B * Lp, qar_block=qblk)
        lws = [LayerWeights(dims, w, k, r, "bf16") for r in range(k)]
        sts = [State(grp.mixers[r], B) for r in range(k)]
        wsp = [grp.mixers[r].workspace(B, Lp) for r in range(k)]
        xp = [to_dev(x, "bf16").view(B * Lp, -1) for _ in range(k)]
        rp = [res.float().cuda().contiguous().view(B * Lp, -1) for _ in range(k)]
        fl = L.SSM_AR2_EXTERNAL if mode == "external" else (L.SSM_AR2_INT8 | L.SSM_QAR_ONESHOT)
        torch.cuda.synchronize()
        grp.run(lambda r, mx, s: mx.prefill(lws[r], sts[r], xp[r], rp[r], flags=fl, workspace=wsp[r], stream=s))
        if mode == "external":
            parts = [rp[r].cpu().numpy().reshape(-1) for r in range(k)]
        else:
            # epochs: AR#1 = 1 (half 1), AR#2 = 2 (half 0): codes at 256, scales at 256 + align256(n)
            for r in range(k):
                codes.append(grp.bufs[r][256:256 + n].cpu().view(torch.int8).numpy())
                so = 256 + (n + 255) // 256 * 256
                scales.append(grp.bufs[r][so:so + 4 * (n // qblk)].cpu().view(torch.float32).numpy())
    for r in range(k):
        q_ref, s_ref = Q.quantize_blocks(parts[r].astype(np.float32), qblk)
        np.testing.assert_array_equal(scales[r], s_ref.reshape(-1))
        np.testing.assert_array_equal(codes[r], q_ref.reshape(-1))


@pytest.mark.parametrize("k,dtype,ar2", [(2, "bf16", "int8"), (4, "bf16", "fp32"), (2, "fp32", "fp32")])
def test_virtual_tp_naive_four_collectives_vs_oracle(k, dtype, ar2):
    """NEXT-3 naive arm (SSM_TP_NAIVE): uniform split of the packed in_proj,
    all-gather of the packed activation and of the conv output, then AR#1 and AR#2 -- four
    collectives per block -- matches the oracle (tp_sim.tp_mixer_forward_naive == mixer_forward)
    and replicates bitwise."""
    dims = MED if dtype == "bf16" else synth.CONFIGS["tiny"]
    flags = (L.SSM_AR2_INT8 if ar2 == "int8" else L.SSM_AR2_FP32) | L.SSM_TP_NAIVE
    L_in, L_out = 24, 3
    outs, w, x, res, grp, sts = _tp_virtual(dims, dtype, k, 2, L_in, L_out, flags, qar_block=min(128, dims.d_model),
                                            naive=True)
    for r in range(1, k):
        assert torch.equal(outs[r], outs[0])
    ref, st_ref = M.mixer_forward(dims, np64(w), x.numpy(), res.numpy())
    resn = res.numpy()
    tol = TOL[dtype] if ar2 != "int8" else TOL["bf16"]
    assert rel(outs[0].double().numpy() - resn, ref - resn) < tol
    h = np.concatenate([sts[r].h.cpu().double().numpy() for r in range(k)], 1)
    assert rel(h, st_ref[1]) < tol
    assert grp.mixers[0].stats()["allreduce"] == 4 * (1 + L_out)     # 2 all-gathers + 2 all-reduces per call


@pytest.mark.parametrize("k", [2, 4, 8])
def test_virtual_qallreduce_requant_bitexact(k):
    """Requantised two-shot (labelled variant, reading Q6): first-stage codes, the shard owners'
    requantised codes/scales and the result equal qar_ref.qallreduce_requant bit for bit; error
    within 2 k max|x| / 254."""
    dims = MED
    n = 6 * dims.d_model * k // 2 * 2
    n -= n % (k * 128)
    parts = synth.partials(k, n, seed=500 + k)
    grp = VirtualGroup(dims, k, "bf16", 64)
    outs = [torch.empty(n, device="cuda") for _ in range(k)]
    dev_parts = [parts[r].cuda() for r in range(k)]
    grp.run(lambda r, mx, s: mx.qallreduce(dev_parts[r], outs[r], stream=s, requant=True))
    ref, codes, scales, q2, s2 = Q.qallreduce_requant(list(parts.numpy()), 128)
    half = ((grp.bufs[0].numel() - 256) // 2) & ~255
    a256 = lambda b: (b + 255) // 256 * 256
    shard = n // k
    for r in range(k):
        base = 256 + half  # epoch 1 -> half 1: codes | scales | shard codes | shard scales
        q = grp.bufs[r][base:base + n].cpu().view(torch.int8).numpy()
        np.testing.assert_array_equal(q, codes[r])
        o2 = base + a256(n) + a256(4 * (n // 128))
        qs = grp.bufs[r][o2:o2 + shard].cpu().view(torch.int8).numpy()
        np.testing.assert_array_equal(qs, q2[r * shard:(r + 1) * shard])
        np.testing.assert_array_equal(outs[r].cpu().numpy(), ref)
    exact = parts.double().sum(0).numpy()
    assert np.all(np.abs(outs[0].cpu().double().numpy() - exact) <= 2 * Q.northstar_bound(list(parts.numpy()), 128) * (1 + 1e-5))


@pytest.mark.parametrize("k", [2, 4])
def test_virtual_tp_mixer_requant_vs_oracle(k):
    outs, w, x, res, grp, sts = _tp_virtual(MED, "bf16", k, 2, 40, 4, L.SSM_AR2_INT8 | L.SSM_QAR_REQUANT)
    for r in range(1, k):
        assert torch.equal(outs[r], outs[0])
    ref, _ = M.mixer_forward(MED, np64(w), x.numpy(), res.numpy())
    resn = res.numpy()
    assert rel(outs[0].double().numpy() - resn, ref - resn) < TOL["bf16"]
