"""bench.py's driver contract on a host without enough GPUs (CPU, no CUDA needed):
* `--gpus N` on a node with fewer devices fails loudly (exit 2, message) instead of timing TP = 1;
* the reference arm (`--impl reference`, the fp64 oracle on the host) prints one JSON line with the
  contract's keys, its own e2e (no host<->device bytes) and a cpu_baseline describing the run."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, cwd=ROOT, env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})


def test_gpus_more_than_devices_fails_loudly():
    r = _run("--gpus", "2", "--steps", "1", "--warmup", "3")
    assert r.returncode == 2
    assert "--gpus 2 but this node has" in r.stderr


def test_reference_arm_json_line():
    r = _run("--impl", "reference", "--config", "tiny", "--steps", "1", "--warmup", "3")
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference"
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["config"]["workload"].startswith("tiny")
