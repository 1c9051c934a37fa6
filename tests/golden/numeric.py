"""Shared definition of the numeric golden fixtures at the benchmarked widths
(test infrastructure: used by ``make_numeric_golden.py`` to write them, by
``tests/test_gpu_numeric_golden.py`` and ``__graft_entry__.smoke()`` to
check the bf16 B200 train step against them).

A fixture holds, for one (model width, reduced depth, schedule, partition)
case, the float64 oracle's ``run_schedule_numeric`` result
(``oracle/gpt_oracle.py``) on seeded inputs:

  * the N per-micro-batch losses;
  * per parameter tensor: the replica-mean gradient's norm and a 64-bucket
    count sketch of it, and the same for the AdamW update (master after -
    master before); 1-D tensors (biases, LayerNorm) are stored in full.

A count sketch S is linear with E||S(e)||^2 = ||e||^2, so
||S(ours) - S(ref)|| / ||S(ref)|| estimates the relative L2 error of the
whole tensor (64 buckets: about +-18 % on the estimate itself).  The hash is
plain integer arithmetic, identical on every host.
"""
from __future__ import annotations

import dataclasses
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
K_SKETCH = 64
LR, WD = 1e-3, 0.01
PARAM_SEED, DATA_SEED = 7, 11


def case_specs():
    """name -> (base config, layers, D, N): BitPipe with the paper-policy
    order and the cost-balanced partition."""
    return {
        # GPT-1.3B width: h 2048, 16 heads of 128, s 2048, V 50304, causal
        "gpt-1.3b-L4": ("gpt-1.3b", 4, 4, 8),
        # BERT-large width: h 1024, 16 heads of 64, s 512, B 4, V 30528, bidirectional
        "bert-large-L4": ("bert-large", 4, 4, 8),
        # GPT-10B width: h 4096, 32 heads of 128, s 2048, V 50304, causal (one layer)
        "gpt-10b-L1": ("gpt-10b", 1, 2, 4),
    }


def case(name):
    """(ModelConfig, Schedule, partition counts) of a fixture case: the
    reduced-depth model at full width, BitPipe with the F2 paper-gate order
    and the cost-balanced partition -- the benchmark's choices."""
    from paper_2410_19367_b200 import schedule as ps
    from paper_2410_19367_b200.model import CONFIGS, balanced_counts
    base, layers, D, N = case_specs()[name]
    cfg = dataclasses.replace(CONFIGS[base], name=f"{CONFIGS[base].name}-L{layers}", layers=layers)
    sched = ps.build_bitpipe(D, N, 2, policy=ps.paper_policy(D))
    return cfg, sched, balanced_counts(cfg, sched)


def path(name):
    return os.path.join(HERE, f"numeric_{name}.pt")


def _mix(idx: torch.Tensor) -> torch.Tensor:
    h = (idx * 2654435761) % (1 << 32)
    h = h ^ (h >> 16)
    h = (h * 0x45D9F3B) % (1 << 32)
    return h ^ (h >> 16)


def sketch(t: torch.Tensor, k: int = K_SKETCH) -> torch.Tensor:
    """Count sketch of a tensor (flattened, float64): bucket and sign of
    element i from an integer hash of i."""
    flat = t.detach().reshape(-1).to("cpu", torch.float64)
    out = torch.zeros(k, dtype=torch.float64)
    step = 1 << 22
    for s in range(0, flat.numel(), step):
        idx = torch.arange(s, min(s + step, flat.numel()), dtype=torch.int64)
        h = _mix(idx)
        sign = 1.0 - 2.0 * ((h >> 20) & 1).to(torch.float64)
        out.index_add_(0, h % k, flat[s:s + idx.numel()] * sign)
    return out


def summarize(tensors: dict) -> dict:
    """{name: {"norm", "sketch", ["full"]}} of a parameter-shaped dict."""
    out = {}
    for k, t in tensors.items():
        t64 = t.detach().to("cpu", torch.float64)
        e = {"norm": t64.norm().item(), "sketch": sketch(t64)}
        if t64.dim() == 1:
            e["full"] = t64.float().clone()
        out[k] = e
    return out


def compare(ours: dict, ref: dict) -> dict:
    """{name: estimated relative L2 error} (exact for stored 1-D tensors)."""
    errs = {}
    for k, r in ref.items():
        o = ours[k]
        if "full" in r:
            errs[k] = ((o["full"].double() - r["full"].double()).norm() / r["full"].double().norm().clamp_min(1e-30)).item()
        else:
            errs[k] = ((o["sketch"] - r["sketch"]).norm() / r["sketch"].norm().clamp_min(1e-30)).item()
    return errs


def load(name):
    return torch.load(path(name), weights_only=False)


def run_b200_step(name, device="cuda:0"):
    """One bf16 train step of the case on the B200 through the product
    Trainer (tcgen05 GEMMs / attention, deferred combined wgrads, fused
    replica-mean AdamW); returns (losses, grad summary, update summary,
    trainer, raw) with raw = (initial params, replica-mean grads, master
    after the update) as host tensors."""
    from paper_2410_19367_b200.model import OptimConfig, init_params, synthetic_batch
    from paper_2410_19367_b200.runtime.executor import Trainer
    cfg, sched, counts = case(name)
    params = init_params(cfg, PARAM_SEED, perturb=True)
    tok, tgt = synthetic_batch(cfg, sched.N, seed=DATA_SEED)
    tr = Trainer(cfg, sched, dtype=torch.bfloat16, optim=OptimConfig(lr=LR, weight_decay=WD), params=params,
                 partition=counts, device=device)
    out = tr.train_step(tok.int().to(device), tgt.int().to(device))
    losses = out.losses.double().cpu()
    g = tr.mean_grads()
    grads = summarize(g)
    master = tr.gather("master")
    upd = summarize({k: master[k].double() - params[k].double() for k in params})
    return losses, grads, upd, tr, (params, g, master)


def adamw_first_step(p0: torch.Tensor, g: torch.Tensor, opt) -> torch.Tensor:
    """float64 AdamW update of the first step (torch.optim.AdamW formula)."""
    g = g.double()
    m = (1 - opt.beta1) * g
    v = (1 - opt.beta2) * g * g
    upd = (m / (1 - opt.beta1)) / (torch.sqrt(v / (1 - opt.beta2)) + opt.eps) + opt.weight_decay * p0.double()
    return -opt.lr * upd
