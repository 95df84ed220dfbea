"""CPU oracle for the tensor-parallel selective-SSM (Mamba) mixer.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product (``paper_2602_21144_b200``) never imports it and has no
CPU fallback.

Plain numpy float64, written from PAPER.md §2.2 / §4 (arXiv 2602.21144) and,
for interfaces and conventions the paper leaves open, SPEC.md and the
readings listed in DESIGN.md §Readings.  It shares no code with the CUDA path.

Modules:
  mixer_ref  single-rank mixer: in_proj, causal conv + SiLU, x_proj, dt/B/C
             split, softplus, ZOH/Euler discretisation, sequential scan, gate,
             out_proj, residual add; prefill/decode with the SSM cache.
  qar_ref    int8 per-block quantised all-reduce, bit-exact codes in fp32,
             with its closed-form error bound.
  tp_sim     channel splitter + the two-all-reduce TP mixer, ranks simulated
             in-process.

  agreement_ref  Table 1's agreement metrics, straight-line.
  attention_ref  Zamba's shared attention + MLP block with its KV cache and TP split (NEXT-1).
  mamba2_ref     the Mamba-2 (SSD) mixer as a per-timestep recurrence, with its TP split (NEXT-4).

Pins (tests/test_oracle_*.py): SPEC.md worked examples (closed forms),
scipy.signal.lfilter on constant-parameter scans, torch conv1d, a pure-Python
brute-force recurrence, HF transformers MambaMixer/FalconMambaMixer/
ZambaMambaMixer slow paths in float64, the pre-norm stack (model_forward)
against chained HF MambaBlocks in float64 (eps-sensitive scale), cache/prefix
invariants, the hand-worked int8 blocks (tests/golden/qar_block.txt,
qar_twoshot.txt) and the closed-form bounds' hand values
(tests/golden/qar_bounds.txt: northstar_bound, fp16_error_bound), HF
ZambaAttentionDecoderLayer and Mamba2Mixer.torch_forward in float64 for the NEXT-1 / NEXT-4
modules.
"""
