"""GPT-2-small language model on the SCFA path.

The paper's LM experiment: a nanoGPT-style decoder, 12
blocks, d=768, 12 heads of 64, no dropout, AdamW (lr 1e-3, betas 0.9/0.95,
weight decay 0.1), bf16.  Keys equal the normalised queries in every variant
(shared-QK).  Variants differ only in the attention call:

  "hash"  H-LM: nb hash buckets from angular LSH of the shared keys
          (hash_sparse.py:34-52's argmax of [xR, -xR]); attention through
          hash_sparse_attention_autograd on the tcgen05 kernels.
  "dense" F-LM: dense causal attention on the same kernels (dense.py:33-93).
  "sdpa"  F-LM on torch's fused SDPA (cuDNN / flash) — a library comparator, and
          the only variant that also runs on CPU (host-logic tests).

The LSH projections R are per layer and per head, drawn once at init and kept
on the device; buckets are recomputed every step from the current keys (they
are not differentiable).  The reference package has no model;
this module is the consumer the path exists for.
"""

import math
from dataclasses import dataclass

import torch
import torch.nn as nn
import torch.nn.functional as F

__all__ = ["LMConfig", "GPT", "make_optimizer", "train_step"]


@dataclass
class LMConfig:
    vocab_size: int = 50304
    block_size: int = 8192
    n_layer: int = 12
    n_head: int = 12
    n_embd: int = 768
    attention: str = "hash"  # "hash" | "dense" | "sdpa"
    n_buckets: int = 16
    exclude_self: bool = False
    seed: int = 0


def lsh_bucket_ids(k, R):
    """Bucket ids (B, T, H) int64 of keys k (B, T, H, D) under projections R (H, D, nb/2).

    argmax of [kR, -kR] with first-max ties (np.argmax order, hash_sparse.py:47-51).  On
    the GPU this is the scfa_lsh_buckets kernel (float64, R shared by the batch); the
    torch expression serves the CPU host-logic tests.
    """
    if k.is_cuda:
        from . import _lib

        B, T, H, D = k.shape
        Rb = R.to(torch.float64).unsqueeze(0).expand(B, *R.shape).contiguous()
        out = torch.empty((B, T, H), dtype=torch.int64, device=k.device)
        dt = _lib.DT_BF16 if k.dtype == torch.bfloat16 else _lib.dtype_code(k)
        kk = k if k.dtype in (torch.bfloat16, torch.float32, torch.float64) else k.float()
        _lib.call("scfa_lsh_buckets", _lib.ptr(kk), dt, B, T, H, D, *kk.stride(), _lib.ptr(Rb), 2 * R.shape[-1],
                  _lib.ptr(out), *out.stride(), _lib.stream_ptr(k.device))
        return out
    with torch.autocast(k.device.type, enabled=False):
        rot = torch.einsum("bthd,hdn->bthn", k.float(), R)
    return torch.cat([rot, -rot], dim=-1).argmax(dim=-1)


class CausalSelfAttention(nn.Module):
    def __init__(self, cfg, layer):
        super().__init__()
        if cfg.n_embd % cfg.n_head:
            raise ValueError("n_embd must be a multiple of n_head")
        self.cfg = cfg
        self.n_head = cfg.n_head
        self.head_dim = cfg.n_embd // cfg.n_head
        # shared-QK: one projection gives queries (keys are their normalisation) and values
        self.c_attn = nn.Linear(cfg.n_embd, 2 * cfg.n_embd, bias=False)
        self.c_proj = nn.Linear(cfg.n_embd, cfg.n_embd, bias=False)
        if cfg.attention == "hash":
            if cfg.n_buckets < 2 or cfg.n_buckets % 2:
                raise ValueError("n_buckets must be even and >= 2")
            g = torch.Generator().manual_seed(cfg.seed * 1000003 + layer)
            R = torch.randn(cfg.n_head, self.head_dim, cfg.n_buckets // 2, generator=g)
            self.register_buffer("R", R, persistent=True)
        elif cfg.attention not in ("dense", "sdpa"):
            raise ValueError(f"unknown attention {cfg.attention!r}")

    def forward(self, x):
        B, T, C = x.shape
        H, D = self.n_head, self.head_dim
        q, v = self.c_attn(x).split(C, dim=2)
        q = q.reshape(B, T, H, D)
        v = v.reshape(B, T, H, D)
        k = F.normalize(q, dim=-1)
        kind = self.cfg.attention
        if kind == "hash":
            from .autograd import hash_sparse_attention_autograd

            with torch.no_grad():
                ids = lsh_bucket_ids(k, self.R)
            y = hash_sparse_attention_autograd(q.contiguous(), k.contiguous(), v.contiguous(), ids, ids,
                                               exclude_self=self.cfg.exclude_self, check=False)
        elif kind == "dense":
            from .autograd import dense_causal_attention_autograd

            y = dense_causal_attention_autograd(q.contiguous(), k.contiguous(), v.contiguous())
        else:
            y = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2),
                                               is_causal=True).transpose(1, 2)
        return self.c_proj(y.reshape(B, T, C))


class MLP(nn.Module):
    def __init__(self, cfg):
        super().__init__()
        self.c_fc = nn.Linear(cfg.n_embd, 4 * cfg.n_embd, bias=False)
        self.c_proj = nn.Linear(4 * cfg.n_embd, cfg.n_embd, bias=False)

    def forward(self, x):
        return self.c_proj(F.gelu(self.c_fc(x), approximate="tanh"))


class Block(nn.Module):
    def __init__(self, cfg, layer):
        super().__init__()
        self.ln_1 = nn.LayerNorm(cfg.n_embd)
        self.attn = CausalSelfAttention(cfg, layer)
        self.ln_2 = nn.LayerNorm(cfg.n_embd)
        self.mlp = MLP(cfg)

    def forward(self, x):
        x = x + self.attn(self.ln_1(x))
        return x + self.mlp(self.ln_2(x))


class GPT(nn.Module):
    def __init__(self, cfg):
        super().__init__()
        self.cfg = cfg
        self.wte = nn.Embedding(cfg.vocab_size, cfg.n_embd)
        self.wpe = nn.Embedding(cfg.block_size, cfg.n_embd)
        self.blocks = nn.ModuleList(Block(cfg, i) for i in range(cfg.n_layer))
        self.ln_f = nn.LayerNorm(cfg.n_embd)
        self.lm_head = nn.Linear(cfg.n_embd, cfg.vocab_size, bias=False)
        self.lm_head.weight = self.wte.weight  # tied, as nanoGPT
        g = torch.Generator().manual_seed(cfg.seed)
        for name, p in self.named_parameters():
            if p.dim() == 2:
                std = 0.02 / math.sqrt(2 * cfg.n_layer) if name.endswith("c_proj.weight") else 0.02
                with torch.no_grad():
                    p.copy_(torch.randn(p.shape, generator=g) * std)

    def n_params(self):
        return sum(p.numel() for p in self.parameters())

    def forward(self, idx, targets=None):
        B, T = idx.shape
        if T > self.cfg.block_size:
            raise ValueError(f"sequence length {T} > block_size {self.cfg.block_size}")
        pos = torch.arange(T, device=idx.device)
        x = self.wte(idx) + self.wpe(pos)
        for blk in self.blocks:
            x = blk(x)
        logits = self.lm_head(self.ln_f(x))
        if targets is None:
            return logits
        return F.cross_entropy(logits.float().view(-1, logits.size(-1)), targets.view(-1))


def make_optimizer(model, lr=1e-3, weight_decay=0.1, betas=(0.9, 0.95)):
    """AdamW with the paper's hyper-parameters; decay on matrices only."""
    decay = [p for p in model.parameters() if p.dim() >= 2]
    other = [p for p in model.parameters() if p.dim() < 2]
    fused = all(p.is_cuda for p in model.parameters())
    return torch.optim.AdamW([{"params": decay, "weight_decay": weight_decay}, {"params": other, "weight_decay": 0.0}],
                             lr=lr, betas=betas, fused=fused)


def train_step(model, opt, idx, targets):
    """One optimiser step: bf16 autocast forward, backward, AdamW.  Returns the loss tensor."""
    dev_type = "cuda" if idx.is_cuda else "cpu"
    with torch.autocast(dev_type, dtype=torch.bfloat16):
        loss = model(idx, targets)
    loss.backward()
    opt.step()
    opt.zero_grad(set_to_none=True)
    return loss.detach()
