"""Greedy generation harness for the agreement study (PAPER.md:591-610
§5.4 Table 1): token embedding -> n_layers x [pre-norm RMSNorm -> TP mixer ->
fp32 residual] -> final RMSNorm -> tied LM head, greedy argmax (lowest index on ties).

The mixer stack runs through libssmtp on k TP ranks -- real NVLink ranks are not available in
this harness, so k > 1 uses virtual ranks on one GPU (virtual.py), which run the same
peer-to-peer all-reduce kernels.  The embedding gather and the LM-head matmul are harness
plumbing outside the §8 hot path (torch).  Weights are seeded synthetic (no checkpoints), so the
agreement numbers measure how much each all-reduce arm perturbs the next-token ranking of a
random-weight model, not a trained model's accuracy."""
from __future__ import annotations

import torch

from . import _lib as L
from .mixer import LayerWeights, TPMixer
from .stack import MixerStack, synthetic_layer
from .virtual import VirtualGroup


class TPLanguageModel:
    def __init__(self, dims, layers_full, emb, k, flags, batch, max_prompt, norm_eps=1e-5, head=None):
        """layers_full: list of full (unsharded) layer weight dicts on the device (synthetic_layer);
        emb: [vocab, d_model] bf16 on the device (input embedding; also the LM head unless `head`)."""
        self.dims, self.k, self.batch, self.eps, self.emb = dims, k, batch, norm_eps, emb
        self.w_head = (emb if head is None else head).float()  # fp32 logits: no bf16 ties in the rankings
        if k > 1:
            self.grp = VirtualGroup(dims, k, "bf16", batch * max_prompt)
            mixers = self.grp.mixers
        else:
            self.grp = None
            mixers = [TPMixer(dims, "bf16")]
        self.mixers = mixers
        self.stacks = [MixerStack(mixers[r], [LayerWeights(dims, w, k, r, "bf16") for w in layers_full], batch,
                                  max_prompt, flags, norm_eps) for r in range(k)]
        self.xh = torch.empty(batch, dims.d_model, dtype=torch.bfloat16, device="cuda")

    def _run(self, fn):
        if self.grp is not None:
            self.grp.run(fn)
        else:
            fn(0, self.mixers[0], torch.cuda.current_stream())
            torch.cuda.synchronize()

    def head(self, res):
        """res [B, D] fp32 -> logits [B, vocab] fp32: final RMSNorm (library kernel) + LM head."""
        self.mixers[0].rmsnorm(res, self.xh, None, self.eps)
        return self.xh.float() @ self.w_head.T

    def generate(self, prompt, n_out, forced=None):
        """prompt [B, L] int64 (device); returns (tokens [B, n_out], logits [n_out, B, vocab] on the
        host).  logits[j] predicts token j; with `forced` [B, n_out], token j fed to the next step is
        forced[:, j] (teacher forcing, so every arm is scored on the same positions)."""
        B, Lp = prompt.shape
        D = self.dims.d_model
        for st in self.stacks:
            st.reset()
        res = [self.emb[prompt].float().reshape(B * Lp, D).contiguous() for _ in range(self.k)]
        self._run(lambda r, mx, s: self.stacks[r].prefill_chunk(res[r], s))
        toks, logits = [], []
        cur = res[0].view(B, Lp, D)[:, -1].contiguous()
        rt = [torch.empty(B, D, device="cuda") for _ in range(self.k)]
        for j in range(n_out):
            lg = self.head(cur)
            logits.append(lg.cpu())
            tok = torch.argmax(lg, dim=-1)            # first maximal index: lowest-index tie-break
            toks.append(tok)
            if j + 1 == n_out:
                break
            feed = forced[:, j] if forced is not None else tok
            x = self.emb[feed].float()
            for r in range(self.k):
                rt[r].copy_(x)
            torch.cuda.synchronize()
            self._run(lambda r, mx, s: self.stacks[r].decode_step(rt[r], s))
            cur = rt[0]
        return torch.stack(toks, 1), torch.stack(logits, 0)


def agreement_study(dims, n_layers, vocab, k_list, batch, prompt_len, n_out, seed=0, arms=("int8", "fp16", "bf16")):
    """Reference arm: exact fp32 all-reduce at each k (and TP=1).  Every arm is teacher-forced with
    the reference arm's tokens; returns a list of result dicts."""
    from .agreement import topk_agreement
    flags = {"fp32": L.SSM_AR2_FP32, "int8": L.SSM_AR2_INT8, "fp16": L.SSM_AR2_FP16, "bf16": L.SSM_AR2_BF16}
    layers = [synthetic_layer(dims, l) for l in range(n_layers)]
    g = torch.Generator(device="cuda").manual_seed(seed)
    emb = torch.randn(vocab, dims.d_model, generator=g, device="cuda").to(torch.bfloat16)
    # untied head: with tied weights a random model's logits are dominated by the current token's
    # own embedding (huge top-1 margin), which no all-reduce perturbation can flip
    head = (torch.randn(vocab, dims.d_model, generator=g, device="cuda") / dims.d_model ** 0.5).to(torch.bfloat16)
    prompt = torch.randint(0, vocab, (batch, prompt_len), generator=g, device="cuda")
    out = []

    def dev(a, b):  # normwise logit deviation and the mean top-1 margin of the reference
        a = a.reshape(-1, vocab).double()
        b = b.reshape(-1, vocab).double()
        t2 = torch.topk(a, 2, dim=-1).values
        return dict(logit_rel_dev=float((a - b).abs().max() / a.abs().max()),
                    ref_top1_margin_over_dev=float((t2[:, 0] - t2[:, 1]).median() / max((a - b).abs().max(), 1e-30)))
    tp1 = TPLanguageModel(dims, layers, emb, 1, 0, batch, prompt_len, head=head)
    tok1, lg1 = tp1.generate(prompt, n_out)
    del tp1
    for k in k_list:
        ref = TPLanguageModel(dims, layers, emb, k, flags["fp32"], batch, prompt_len, head=head)
        tok_r, lg_r = ref.generate(prompt, n_out, forced=tok1)
        del ref
        m = topk_agreement(lg1.reshape(-1, vocab).numpy(), lg_r.reshape(-1, vocab).numpy())
        out.append(dict(k=k, arm="fp32", vs="tp1", **m, **dev(lg1, lg_r)))
        for arm in arms:
            mdl = TPLanguageModel(dims, layers, emb, k, flags[arm], batch, prompt_len, head=head)
            _, lg = mdl.generate(prompt, n_out, forced=tok1)
            del mdl
            m = topk_agreement(lg_r.reshape(-1, vocab).numpy(), lg.reshape(-1, vocab).numpy())
            out.append(dict(k=k, arm=arm, vs=f"tp{k}_fp32", **m, **dev(lg_r, lg)))
        torch.cuda.empty_cache()
    return out
