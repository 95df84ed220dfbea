"""Bench lines for every BASELINE config on one GPU (TP = 1), appended to a JSONL file:
cfg1 tiny fp32 latency, cfg2 Mamba-2.8B (default), cfg3 Falcon-Mamba-7B, cfg4 Zamba-7B hybrid,
cfg5 Mamba-2.8B long-context TTFT sweep (16K / 32K / 64K prompt, batch 8), and Mamba-2 2.7B.

    python scripts/config_sweep.py OUT.jsonl
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUNS = [
    ("tiny", ["--config", "tiny", "--steps", "20", "--warmup", "5", "--no-cpu"]),
    ("falcon7b", ["--config", "falcon7b", "--steps", "1", "--warmup", "1", "--no-cpu", "--no-e2e"]),
    ("zamba7b", ["--config", "zamba7b", "--steps", "1", "--warmup", "1", "--no-cpu", "--no-e2e"]),
    ("long16k", ["--config", "mamba2.8b-long", "--prompt", "16384", "--steps", "1", "--warmup", "1", "--no-cpu", "--no-e2e"]),
    ("long32k", ["--config", "mamba2.8b-long", "--prompt", "32768", "--steps", "1", "--warmup", "1", "--no-cpu", "--no-e2e"]),
    ("long64k", ["--config", "mamba2.8b-long", "--steps", "1", "--warmup", "1", "--no-cpu", "--no-e2e"]),
    ("mamba2", ["--config", "mamba2-2.7b", "--steps", "1", "--warmup", "1", "--no-cpu", "--no-e2e"]),
]
out = sys.argv[1]
only = set(sys.argv[2:])
for name, args in RUNS:
    if only and name not in only:
        continue
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=900)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else json.dumps({"error": r.stderr[-400:]})
    with open(out, "a") as f:
        f.write(json.dumps({"run": name, "line": json.loads(line) if line.startswith("{") else line}) + "\n")
    print(name, line[:200], flush=True)
