#!/usr/bin/env python
"""Agreement of the quantised all-reduce arms with the exact one (Table 1
structure) on seeded synthetic Mamba-2.8B-shaped weights, virtual TP ranks on one GPU.
    python scripts/agreement.py [--layers 8] [--k 2 4 8] [--batch 16] [--prompt 256] [--out 64]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_21144_b200.generate import agreement_study  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="mamba2.8b")
p.add_argument("--layers", type=int, default=64)
p.add_argument("--vocab", type=int, default=50280)   # Mamba's GPT-NeoX vocabulary size (HF MambaConfig)
p.add_argument("--k", type=int, nargs="+", default=[2, 4, 8])
p.add_argument("--batch", type=int, default=16)
p.add_argument("--prompt", type=int, default=256)
p.add_argument("--out", type=int, default=64)
a = p.parse_args()
dims = synth.CONFIGS[a.config]
for r in agreement_study(dims, a.layers, a.vocab, a.k, a.batch, a.prompt, a.out):
    r.update(config=a.config, layers=a.layers, vocab=a.vocab, batch=a.batch, prompt=a.prompt, positions=a.batch * a.out)
    print(json.dumps(r), flush=True)
