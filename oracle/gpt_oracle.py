"""TEST INFRASTRUCTURE ONLY -- CPU oracle of the BitPipe train step.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module, and only as the checker / the timed CPU
baseline.  The product path never calls it.

What it restates
----------------
The reference has no numeric train step; it exists only as the SPEC
``runtime`` module (reference ``SPEC.md:408-468``):

  * ``run_schedule_numeric(schedule, model, batch, seed)``:
    one worker per device executes its task list in order; activations and
    gradients flow along schedule edges (F(m,s-1)->F(m,s), F(m,last)->B(m,
    last), B(m,s+1)->B(m,s), reference ``schedules.py:181-199``); gradients
    accumulate over micro-batches; bidirectional runs hold two identically
    initialised replicas whose gradients are averaged before
    ONE optimizer update after the flush;
  * ``sequential_baseline(model, batch, seed)``: one worker,
    mean over the N micro-batches, one update.  Schedule independence
     says both must agree.

The schedule is consumed in the reference's wire format (the JSON of
``pipesched.schedules.dump_schedule``, reference ``schedules.py:301-356``);
the golden dumps in ``tests/golden/`` come from the reference itself.

Model (the SPEC's ToyModel is replaced by the north star's transformer;
choices mirror ``paper_2410_19367_b200/model.py`` and are restated here so
the oracle does not import product code): pre-LN GPT/BERT block, learned
positions, untied LM head, tanh-GELU, mean token cross-entropy per
micro-batch, AdamW (torch.optim.AdamW formula) as the single update.
Arithmetic: float64 by default, float32 optional.

Parity pinning: the schedule orders are pinned to the reference (golden
dumps/hashes).  Numeric values are NOT pinned by the reference (it has no
numeric implementation); they are pinned by this restatement
plus the SPEC's own schedule-independence theorem, which the tests check
(run_schedule_numeric == sequential_baseline for every schedule).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass

import torch

__all__ = ["OracleConfig", "StepResult", "stage_halfblocks", "sequential_baseline", "run_schedule_numeric",
           "execute_orders", "replica_mean_grads", "adamw_update"]


@dataclass(frozen=True)
class OracleConfig:
    layers: int
    hidden: int
    heads: int
    seq: int
    vocab: int
    micro_batch: int
    causal: bool = True
    ln_eps: float = 1e-5
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.0


@dataclass
class StepResult:
    losses: torch.Tensor          # [N] per-micro-batch mean CE, index m-1
    grads: dict                   # synchronised (replica-mean) gradients
    params: dict                  # parameters after the single update
    adam_m: dict
    adam_v: dict


# -- partition (restates the product's rule; tests check they agree) ---------
def stage_halfblocks(layers: int, num_stages: int):
    n = 2 * layers
    base, rem = divmod(n, num_stages)
    extra = [0] * num_stages
    for s in sorted(range(num_stages), key=lambda s: (abs(2 * s - (num_stages - 1)), s))[:rem]:
        extra[s] = 1
    out, start = [], 0
    for s in range(num_stages):
        out.append(list(range(start, start + base + extra[s])))
        start += base + extra[s]
    return out


# -- model pieces (float64 autograd) -------------------------------------------
def _ln(x, w, b, eps):
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    return (x - mu) / torch.sqrt(var + eps) * w + b


def _gelu(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x * x * x)))


def _attn_half(P, l, x, cfg: OracleConfig):
    B, S, h = x.shape
    H, Dh = cfg.heads, h // cfg.heads
    p = f"layers.{l}."
    a = _ln(x, P[p + "ln1.w"], P[p + "ln1.b"], cfg.ln_eps)
    qkv = a @ P[p + "attn.qkv.w"].t() + P[p + "attn.qkv.b"]
    q, k, v = qkv.view(B, S, 3, H, Dh).permute(2, 0, 3, 1, 4)
    s = (q @ k.transpose(-1, -2)) / math.sqrt(Dh)
    if cfg.causal:
        mask = torch.triu(torch.ones(S, S, dtype=torch.bool), 1)
        s = s.masked_fill(mask, float("-inf"))
    o = (s.softmax(-1) @ v).permute(0, 2, 1, 3).reshape(B, S, h)
    return x + o @ P[p + "attn.proj.w"].t() + P[p + "attn.proj.b"]


def _mlp_half(P, l, x, cfg: OracleConfig):
    p = f"layers.{l}."
    m = _ln(x, P[p + "ln2.w"], P[p + "ln2.b"], cfg.ln_eps)
    u = m @ P[p + "mlp.fc1.w"].t() + P[p + "mlp.fc1.b"]
    return x + _gelu(u) @ P[p + "mlp.fc2.w"].t() + P[p + "mlp.fc2.b"]


def _embed(P, tokens):
    S = tokens.shape[1]
    return P["embed.wte"][tokens] + P["embed.wpe"][:S].unsqueeze(0)


def _head_loss(P, x, targets, cfg: OracleConfig):
    xf = _ln(x, P["head.lnf.w"], P["head.lnf.b"], cfg.ln_eps)
    logits = xf @ P["head.lm.w"].t()
    return torch.nn.functional.cross_entropy(logits.reshape(-1, logits.shape[-1]), targets.reshape(-1))


def _run_stage(P, hbs, x, cfg, *, first, last, tokens, targets):
    if first:
        x = _embed(P, tokens)
    for hb in hbs:
        l, half = divmod(hb, 2)
        x = _attn_half(P, l, x, cfg) if half == 0 else _mlp_half(P, l, x, cfg)
    if last:
        return _head_loss(P, x, targets, cfg)
    return x


def _clone_params(params, dtype):
    return {k: v.detach().to(dtype).clone().requires_grad_(True) for k, v in params.items()}


def adamw_update(params, grads, m, v, cfg: OracleConfig, step: int):
    """torch.optim.AdamW step (decoupled weight decay) in the param dtype."""
    newp, newm, newv = {}, {}, {}
    b1, b2 = cfg.beta1, cfg.beta2
    bc1, bc2 = 1 - b1 ** step, 1 - b2 ** step
    for k, p in params.items():
        g = grads[k]
        mk = b1 * m[k] + (1 - b1) * g
        vk = b2 * v[k] + (1 - b2) * g * g
        upd = (mk / bc1) / (torch.sqrt(vk / bc2) + cfg.eps) + cfg.weight_decay * p
        newp[k], newm[k], newv[k] = p - cfg.lr * upd, mk, vk
    return newp, newm, newv


def _zeros_like(params):
    return {k: torch.zeros_like(v) for k, v in params.items()}


def sequential_baseline(cfg: OracleConfig, params: dict, tokens, targets, *, dtype=torch.float64,
                        adam_state=None, step: int = 1) -> StepResult:
    """One worker, N micro-batches, mean loss, one AdamW update."""
    N = tokens.shape[0]
    P = _clone_params(params, dtype)
    losses = torch.zeros(N, dtype=dtype)
    for i in range(N):
        x = _embed(P, tokens[i])
        for hb in range(2 * cfg.layers):
            l, half = divmod(hb, 2)
            x = _attn_half(P, l, x, cfg) if half == 0 else _mlp_half(P, l, x, cfg)
        loss = _head_loss(P, x, targets[i], cfg)
        (loss / N).backward()
        losses[i] = loss.detach()
    grads = {k: p.grad.detach().clone() for k, p in P.items()}
    base = {k: p.detach() for k, p in P.items()}
    m0, v0 = adam_state if adam_state is not None else (_zeros_like(base), _zeros_like(base))
    newp, m1, v1 = adamw_update(base, grads, m0, v0, cfg, step)
    return StepResult(losses, grads, newp, m1, v1)


def execute_orders(sch: dict, replicas: dict, stage_fn, N: int):
    """Message-passing execution of the reference per-device orders (the
    generic core of SPEC ``run_schedule_numeric``), shared
    by the GPT oracle and the SPEC ToyModel (``oracle/toy_model.py``).

    ``replicas``: {direction: {name: leaf tensor requiring grad}}, one per
    stage-map direction.  ``stage_fn(P, stage, x_in, mb)`` runs one stage
    forward of micro-batch ``mb`` (1-based) on replica ``P`` and returns the
    activation (or, on the last stage, the scalar loss).  Each replica
    averages its own N/len(dirs) micro-batches; gradients accumulate in the
    replicas' ``.grad``.  Returns the per-micro-batch losses.

    Workers advance in lock-step rounds: a device runs its next task when
    that task's input message (or micro-batch data) is present, following
    the dataflow edges of reference ``schedules.py:181-199``.  A round in
    which nobody can advance raises RuntimeError (SPEC DeadlockDetected),
    as do messages left over after the flush (SPEC ProtocolViolation).
    """
    D, v = sch["D"], sch["v"]
    S_tot = D * v
    dirs = [m["direction"] for m in sch["stage_maps"]]
    n_rep = N // len(dirs)  # micro-batches per replica
    rows = [[tuple(r[:4]) for r in dev] for dev in sch["per_device"]]
    pos = [0] * D
    acts, grads_in, stash = {}, {}, {}
    losses = [None] * N
    last = S_tot - 1
    remaining = sum(len(r) for r in rows)
    while remaining:
        moved = False
        for d in range(D):
            while pos[d] < len(rows[d]):
                kind, mb, s, dr = rows[d][pos[d]]
                P = replicas[dr]
                if kind == "F":
                    if s > 0 and (dr, mb, s - 1) not in acts:
                        break
                    x_in = None if s == 0 else acts.pop((dr, mb, s - 1)).requires_grad_(True)
                    out = stage_fn(P, s, x_in, mb)
                    stash[(dr, mb, s)] = (x_in, out)
                    if s == last:
                        losses[mb - 1] = out.detach()
                    else:
                        acts[(dr, mb, s)] = out.detach()
                else:
                    if (dr, mb, s) not in stash or (s < last and (dr, mb, s + 1) not in grads_in):
                        break
                    x_in, out = stash.pop((dr, mb, s))
                    if s == last:
                        (out / n_rep).backward()
                    else:
                        out.backward(grads_in.pop((dr, mb, s + 1)))
                    if s > 0:
                        grads_in[(dr, mb, s)] = x_in.grad.detach()
                pos[d] += 1
                remaining -= 1
                moved = True
        if remaining and not moved:
            raise RuntimeError("oracle executor deadlocked: no device can advance")
    if acts or grads_in or stash:
        raise RuntimeError("oracle executor: undelivered messages after flush")
    return torch.stack(losses)


def replica_mean_grads(replicas: dict, names) -> dict:
    """The eager replica-pair all-reduce as a mean: each
    replica averaged its own N/2 micro-batches, so the pair mean is the
    N-micro-batch mean."""
    dirs = list(replicas)
    if len(dirs) == 2:
        return {k: (replicas[dirs[0]][k].grad + replicas[dirs[1]][k].grad) * 0.5 for k in names}
    return {k: replicas[dirs[0]][k].grad.clone() for k in names}


def run_schedule_numeric(cfg: OracleConfig, schedule_json: str | dict, params: dict, tokens, targets, *,
                         dtype=torch.float64, adam_state=None, step: int = 1, halfblocks=None) -> StepResult:
    """SPEC ``run_schedule_numeric`` for the GPT/BERT
    model: execute the reference per-device orders (wire format of
    ``dump_schedule``, reference ``schedules.py:301-356``) with message
    passing (:func:`execute_orders`) on two identically initialised
    replicas, average their gradients, then ONE AdamW update."""
    sch = json.loads(schedule_json) if isinstance(schedule_json, str) else schedule_json
    S_tot = sch["D"] * sch["v"]
    dirs = [m["direction"] for m in sch["stage_maps"]]
    # partition: the uniform rule, or an explicit per-stage half-block list
    # (the product's cost-balanced partition); the result is the same model
    hbs = [list(h) for h in halfblocks] if halfblocks is not None else stage_halfblocks(cfg.layers, S_tot)
    assert len(hbs) == S_tot and [hb for h in hbs for hb in h] == list(range(2 * cfg.layers))
    replicas = {d: _clone_params(params, dtype) for d in dirs}
    last = S_tot - 1

    def stage_fn(P, s, x_in, mb):
        return _run_stage(P, hbs[s], x_in, cfg, first=s == 0, last=s == last,
                          tokens=tokens[mb - 1], targets=targets[mb - 1])

    losses = execute_orders(sch, replicas, stage_fn, tokens.shape[0])
    names = list(params)
    g = replica_mean_grads(replicas, names)
    base = {k: replicas[dirs[0]][k].detach() for k in names}
    m0, v0 = adam_state if adam_state is not None else (_zeros_like(base), _zeros_like(base))
    newp, m1, v1 = adamw_update(base, g, m0, v0, cfg, step)
    return StepResult(losses, g, newp, m1, v1)


def layer_sample_seconds(cfg: OracleConfig, *, dtype=torch.float32, seed: int = 0) -> float:
    """CPU wall time of forward + backward of ONE transformer layer (attention
    half + MLP half) on ONE micro-batch -- the bounded sample the benchmark's
    CPU baseline extrapolates from (uses torch's intra-op threads)."""
    import time as _time
    g = torch.Generator().manual_seed(seed)
    h, f = cfg.hidden, 4 * cfg.hidden
    P = {
        "layers.0.ln1.w": torch.ones(h), "layers.0.ln1.b": torch.zeros(h),
        "layers.0.attn.qkv.w": torch.randn(3 * h, h, generator=g) * 0.02, "layers.0.attn.qkv.b": torch.zeros(3 * h),
        "layers.0.attn.proj.w": torch.randn(h, h, generator=g) * 0.02, "layers.0.attn.proj.b": torch.zeros(h),
        "layers.0.ln2.w": torch.ones(h), "layers.0.ln2.b": torch.zeros(h),
        "layers.0.mlp.fc1.w": torch.randn(f, h, generator=g) * 0.02, "layers.0.mlp.fc1.b": torch.zeros(f),
        "layers.0.mlp.fc2.w": torch.randn(h, f, generator=g) * 0.02, "layers.0.mlp.fc2.b": torch.zeros(h),
    }
    P = {k: v.to(dtype).requires_grad_(True) for k, v in P.items()}
    x = torch.randn(cfg.micro_batch, cfg.seq, h, generator=g).to(dtype).requires_grad_(True)
    t0 = _time.perf_counter()
    y = _mlp_half(P, 0, _attn_half(P, 0, x, cfg), cfg)
    y.backward(torch.ones_like(y))
    return _time.perf_counter() - t0
