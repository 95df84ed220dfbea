"""CPU checks of the C-ABI library: it loads, exports every symbol include/ssm_tp.h
declares, and validates arguments synchronously (no compute calls without a GPU)."""
import ctypes as C
import os
import re

import pytest

import synth
from paper_2602_21144_b200 import _lib as L
from paper_2602_21144_b200 import TPMixer, channel_range, SSMError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "ssm_tp.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^\s*(?:ssm_status_t|const char\*)\s+(ssm_\w+)\s*\(", src, re.M)))


def test_header_symbols_exported():
    names = _declared()
    assert len(names) >= 20
    lib = C.CDLL(L.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/ssm_tp.h but not exported"
    assert set(names) == set(L.EXPORTED)


def test_version_and_last_error():
    assert b"sm_100a" in L.LIB.ssm_version()
    assert isinstance(L.LIB.ssm_last_error(), bytes)


def test_init_validation_errors():
    tiny = synth.CONFIGS["tiny"]
    with pytest.raises(SSMError) as e:
        TPMixer(tiny, "fp32", rank=0, tp_size=3, device="cpu")         # SPEC.md:251 shard error
    assert e.value.name == "SSM_ERR_SHARD"
    fake = [256 * (i + 1) for i in range(4)]
    nbytes = L.comm_bytes(L.make_config(tiny, "fp32", 64), 4, 128)
    with pytest.raises(SSMError) as e:
        TPMixer(tiny, "fp32", rank=4, tp_size=4, peer_bufs=fake, buf_bytes=nbytes, device="cpu")
    assert e.value.name == "SSM_ERR_RANK"
    with pytest.raises(SSMError) as e:
        TPMixer(tiny, "fp32", rank=0, tp_size=16, device="cpu")
    assert e.value.name == "SSM_ERR_UNSUPPORTED"
    with pytest.raises(SSMError) as e:
        TPMixer(tiny, "fp32", rank=0, tp_size=2, peer_bufs=None, device="cpu")
    assert e.value.name == "SSM_ERR_ARG"
    with pytest.raises(SSMError) as e:
        TPMixer(tiny, "fp32", rank=0, tp_size=2, peer_bufs=fake[:2], buf_bytes=64, device="cpu")
    assert e.value.name == "SSM_ERR_ARG"
    bad = synth.MixerDims(d_model=64, d_inner=128, d_state=32, dt_rank=4)
    with pytest.raises(SSMError) as e:
        TPMixer(bad, "fp32", device="cpu")
    assert e.value.name == "SSM_ERR_UNSUPPORTED"
    z = synth.MixerDims(d_model=256, d_inner=512, dt_rank=16, n_heads=2)
    TPMixer(z, "bf16", rank=1, tp_size=4, peer_bufs=fake, buf_bytes=L.comm_bytes(L.make_config(z), 4, 64),
            device="cpu")  # heads split over 2 ranks each: valid


def test_sizes_and_channel_ranges():
    tiny = synth.CONFIGS["tiny"]
    m = TPMixer(tiny, "fp32", device="cpu")
    assert m.workspace_bytes(2, 64) > 2 * 64 * 2 * tiny.d_inner * 4
    assert m.workspace_bytes(0, 0) == 0
    assert channel_range(128, 4, 2) == (64, 96)
    with pytest.raises(SSMError):
        channel_range(100, 3, 0)
    cfg = L.make_config(synth.CONFIGS["mamba2.8b"], "bf16")
    b1 = L.comm_bytes(cfg, 8, 1024)
    b2 = L.comm_bytes(cfg, 8, 2048)
    assert b2 > b1 > 2 * 1024 * 2560          # two halves of at least the fp32 AR#2 payload


def test_state_and_calls_validate_before_touching_the_device():
    tiny = synth.CONFIGS["tiny"]
    m = TPMixer(tiny, "fp32", device="cpu")
    st = C.c_void_p()
    rc = L.LIB.ssm_state_alloc(m.handle, 2, None, 0, None, 0, None, C.byref(st))
    assert L.STATUS[rc] == "SSM_ERR_ARG"
    rc = L.LIB.ssm_mixer_prefill(m.handle, None, None, None, None, 1, 1, 0, None, 0, None)
    assert L.STATUS[rc] == "SSM_ERR_ARG"
    rc = L.LIB.ssm_qallreduce(m.handle, None, None, 128, 0, None)
    assert L.STATUS[rc] == "SSM_ERR_ARG"


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(L, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(ImportError):
        L._load()
