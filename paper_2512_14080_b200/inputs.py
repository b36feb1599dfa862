"""Seeded synthetic inputs shared by the tests, the bench and the oracle legs.

This module holds NONE of the method's arithmetic (no routing, no GEMM, no
activation): it only draws random tensors with the shapes and distributions
stated in DESIGN.md §5 (input recipe).  Router scores S are the caller's
input to ``sonic_route`` (the router GEMM + softmax sit outside the boundary,
P:284 footnote), so they are drawn here as softmax(N(0,1) logits) in fp32.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

# The BASELINE.json configs (T, d, n, E, K).
CONFIGS = {
    "tiny": dict(T=256, d=64, n=32, E=8, K=2),
    "7b": dict(T=32768, d=1536, n=256, E=128, K=8),
    "qwen3": dict(T=32768, d=2048, n=768, E=128, K=8),
    "dsv3": dict(T=65536, d=7168, n=2048, E=256, K=8),
    "kimi": dict(T=65536, d=7168, n=2048, E=384, K=8),
    # the paper's token-rounding speed study (Table 14 / Fig. 12: T, d, n, K = 16384, 1536,
    # 1024, 2 at E = 128): TC vs TR context, not a BASELINE.json config
    "tr_study": dict(T=16384, d=1536, n=1024, E=128, K=2),
}


@dataclass
class MoEInputs:
    X: torch.Tensor    # [T,d] bf16
    W1: torch.Tensor   # [E,d,2n] bf16
    W2: torch.Tensor   # [E,n,d] bf16
    dO: torch.Tensor   # [T,d] bf16
    S: torch.Tensor    # [T,E] fp32 router scores (softmax of logits)


def make_token_inputs(T, d, E, seed=0, device="cpu"):
    """X, dO ~ N(0,1) bf16 and S = softmax(N(0,1) logits) fp32 for T tokens (expert-parallel runs:
    every rank draws its own microbatch)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    X = torch.randn(T, d, generator=g, device=device).to(torch.bfloat16)
    dO = torch.randn(T, d, generator=g, device=device).to(torch.bfloat16)
    S = torch.softmax(torch.randn(T, E, generator=g, device=device), dim=1).contiguous()
    return X.contiguous(), dO.contiguous(), S


def make_expert_weights(e_lo, e_hi, d, n, seed=0, device="cpu"):
    """W1 ~ N(0,1/d), W2 ~ N(0,1/n) (bf16) for experts [e_lo, e_hi); expert e is drawn from its own
    seed, so any sharding of the experts over ranks yields the same weights."""
    W1 = torch.empty(e_hi - e_lo, d, 2 * n, dtype=torch.bfloat16, device=device)
    W2 = torch.empty(e_hi - e_lo, n, d, dtype=torch.bfloat16, device=device)
    g = torch.Generator(device=device)
    for i, e in enumerate(range(e_lo, e_hi)):
        g.manual_seed(seed * 100003 + e)
        W1[i] = (torch.randn(d, 2 * n, generator=g, device=device) / math.sqrt(d)).to(torch.bfloat16)
        W2[i] = (torch.randn(n, d, generator=g, device=device) / math.sqrt(n)).to(torch.bfloat16)
    return W1, W2


def make_inputs(T, d, n, E, K=None, seed=0, device="cpu", skew=0.0, tie_levels=0):
    """X ~ N(0,1); W1 ~ N(0,1/d); W2 ~ N(0,1/n); dO ~ N(0,1); logits ~ N(0,1).

    skew > 0 adds a per-expert bias skew*N(0,1) to the logits (skewed load).
    tie_levels > 0 quantises the logits to that many levels so that exact
    score ties occur (tie-break tests).
    """
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    bf = torch.bfloat16
    X = torch.randn(T, d, generator=g, device=device).to(bf)
    W1 = (torch.randn(E, d, 2 * n, generator=g, device=device) / math.sqrt(d)).to(bf)
    W2 = (torch.randn(E, n, d, generator=g, device=device) / math.sqrt(n)).to(bf)
    dO = torch.randn(T, d, generator=g, device=device).to(bf)
    logits = torch.randn(T, E, generator=g, device=device)
    if skew:
        logits = logits + skew * torch.randn(1, E, generator=g, device=device)
    if tie_levels:
        logits = torch.round(logits * tie_levels) / tie_levels
    S = torch.softmax(logits.float(), dim=1).contiguous()
    return MoEInputs(X.contiguous(), W1.contiguous(), W2.contiguous(), dO.contiguous(), S)
