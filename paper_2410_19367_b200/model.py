"""Model family, parameter layout and the layer -> virtual-stage partitioner.

The reference has no layer partitioner (SPEC.md:219 lists it as a non-goal)
and no model: its train step is specified on a toy MLP.
The north star fixes the model family instead: a GPT-style (causal) or
BERT-style (bidirectional attention) pre-LN transformer.  Choices, stated
once here and restated in ``oracle/gpt_oracle.py``:

  * learned token + position embeddings; untied LM head (no bias);
  * pre-LN blocks: x += proj(attn(LN1 x)); x += fc2(gelu_tanh(fc1(LN2 x)));
    FFN = 4h; final LN before the head;
  * loss = mean token cross-entropy per micro-batch; the step objective is
    the mean over the N micro-batches (each replica averages its own N/2,
    the replica pair averages);
  * init: N(0, 0.02) weights, output projections N(0, 0.02/sqrt(2L)),
    zero biases, unit LN gains (``perturb=True`` adds small noise to biases
    and LN params so parity tests exercise every gradient).

Partition: the 2L half-blocks (attention half, MLP half)
are split over the v*D virtual stages of one direction in contiguous runs;
stage 0 additionally owns the embedding and stage v*D-1 the final LN, LM
head and loss.  In the V map both sit on device 0 (down) / D-1 (up).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

__all__ = ["ModelConfig", "CONFIGS", "StagePlan", "stage_partition", "balanced_counts", "stage_costs",
           "fit_task_costs", "modelled_task_times", "calibrated_counts", "load_calibration", "resolve_partition",
           "device_loads", "param_specs", "stage_param_names",
           "init_params", "flops_per_token"]


@dataclass(frozen=True)
class ModelConfig:
    name: str
    layers: int
    hidden: int
    heads: int
    seq: int
    vocab: int
    micro_batch: int = 1
    causal: bool = True
    ffn_mult: int = 4
    ln_eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    @property
    def ffn(self) -> int:
        return self.ffn_mult * self.hidden

    @property
    def tokens_per_microbatch(self) -> int:
        return self.micro_batch * self.seq

    def n_params(self) -> int:
        return sum(math.prod(s) for _, s, _ in param_specs(self))


CONFIGS = {
    # BASELINE.json configs (SURVEY §8(d) hyper-parameters)
    "tiny": ModelConfig("tiny-gpt", layers=4, hidden=64, heads=4, seq=32, vocab=256, micro_batch=2),
    "bert-large": ModelConfig("bert-large", layers=24, hidden=1024, heads=16, seq=512, vocab=30528,
                              micro_batch=4, causal=False),
    "gpt-1.3b": ModelConfig("gpt-1.3b", layers=24, hidden=2048, heads=16, seq=2048, vocab=50304, micro_batch=1),
    "gpt-10b": ModelConfig("gpt-10b", layers=48, hidden=4096, heads=32, seq=2048, vocab=50304, micro_batch=1),
    # small configs used by tests
    "small": ModelConfig("small-gpt", layers=4, hidden=256, heads=4, seq=128, vocab=512, micro_batch=2),
    "small-bert": ModelConfig("small-bert", layers=2, hidden=128, heads=2, seq=128, vocab=300, micro_batch=2,
                              causal=False),
}


def flops_per_token(cfg: ModelConfig) -> float:
    """Megatron convention, no recompute, full (non-causal-discounted)
    attention: 3 * (24 L h^2 + 4 s L h + 2 V h)."""
    L, h, s, V = cfg.layers, cfg.hidden, cfg.seq, cfg.vocab
    return 3.0 * (24 * L * h * h + 4 * s * L * h + 2 * V * h)


@dataclass(frozen=True)
class StagePlan:
    stage: int
    halfblocks: tuple[int, ...]   # hb = 2*layer (+1 for the MLP half)
    embed: bool
    head: bool


def stage_partition(cfg: ModelConfig, num_stages: int, counts=None) -> tuple[StagePlan, ...]:
    """Contiguous split of the 2L half-blocks over ``num_stages`` stages.

    Default (uniform): remainders go to the middle stages first (the end
    stages already carry the embedding / LM head).  ``counts`` gives the
    number of half-blocks per stage explicitly (e.g. :func:`balanced_counts`).
    Every stage gets >= 0 half-blocks; stages with none still pass
    activations through (and own embed/head if ends).
    """
    n = 2 * cfg.layers
    if counts is None:
        base, rem = divmod(n, num_stages)
        extra = [0] * num_stages
        order = sorted(range(num_stages), key=lambda s: (abs(2 * s - (num_stages - 1)), s))
        for s in order[:rem]:
            extra[s] = 1
        counts = [base + e for e in extra]
    counts = [int(c) for c in counts]
    if len(counts) != num_stages or min(counts) < 0 or sum(counts) != n:
        raise ValueError(f"partition counts {counts} do not split {n} half-blocks over {num_stages} stages")
    plans, start = [], 0
    for s in range(num_stages):
        plans.append(StagePlan(s, tuple(range(start, start + counts[s])), s == 0, s == num_stages - 1))
        start += counts[s]
    return tuple(plans)


# Cost model of the partitioner, in GEMM-equivalent FLOPs per token,
# calibrated on B200 (tools/stage_times.py, GPT-1.3B D=8: attention half :
# MLP half : LM head = 1 : 1 : 2.9 in measured task time, B / F = 1.98):
# attention-core FLOPs run at ~0.45x the GEMMs' rate, the LM-head GEMMs
# (N = V) at ~1.5x, and the fused cross-entropy moves 3 V 2-byte values per
# token at HBM speed (~6.5 TB/s vs ~1 PFLOP/s of GEMM).
ATTN_CORE_WEIGHT = 2.3
HEAD_GEMM_WEIGHT = 0.6
XENT_FLOPS_PER_BYTE = 1000.0 / 6.5


def _hb_flops(cfg: ModelConfig, hb: int) -> float:
    """Forward cost per token of half-block ``hb`` (attention or MLP half)."""
    h, s = cfg.hidden, cfg.seq
    if hb % 2 == 0:  # QKV + out-projection GEMMs, attention scores / context
        return 8.0 * h * h + ATTN_CORE_WEIGHT * 4.0 * s * h * (0.5 if cfg.causal else 1.0)
    return 4.0 * h * cfg.ffn  # fc1 + fc2


def stage_costs(cfg: ModelConfig, counts) -> list[float]:
    """Forward cost per token of each stage (see the cost-model constants):
    its half-blocks plus, on the last stage, the LM head and the fused
    softmax cross-entropy; the embedding gather is free."""
    out, start = [], 0
    for s, c in enumerate(counts):
        f = sum(_hb_flops(cfg, hb) for hb in range(start, start + c))
        if s == len(counts) - 1:
            f += HEAD_GEMM_WEIGHT * 2.0 * cfg.vocab * cfg.hidden + XENT_FLOPS_PER_BYTE * 3 * cfg.vocab * 2
        out.append(f)
        start += c
    return out


def device_loads(cfg: ModelConfig, counts, stage_maps) -> list[float]:
    """Per-device compute of one direction-symmetric partition: every
    direction's stage map places the same stages (same partition, one model
    replica per direction) on its devices (schedules.py:58-108 StageMap)."""
    cost = stage_costs(cfg, counts)
    D = max(max(m.assignment) for m in stage_maps) + 1
    loads = [0.0] * D
    for m in stage_maps:
        for st, d in enumerate(m.assignment):
            loads[d] += cost[st]
    return loads


def balanced_counts(cfg: ModelConfig, schedule) -> list[int]:
    """Half-blocks per stage for a cost-balanced partition (SURVEY §7 step
    3): the stage that also computes the LM head (~2 V h FLOPs per token,
    3-4 half-blocks at GPT sizes) gets fewer half-blocks.

    Objective: the makespan of the reference ASAP replay (``list_schedule``,
    fusion.py:34-77) of ``schedule``'s fixed per-device orders with task
    durations F = stage FLOPs, B = 2 x F (one GPU per logical device, free
    communication), then the most loaded device, then the spread of device
    loads.  Local search from the uniform split, moving one half-block
    across a stage boundary at a time while the objective improves; the
    result depends only on (cfg, schedule) and is deterministic."""
    from fractions import Fraction

    from .schedule import list_schedule

    S = schedule.num_stages
    maps = [schedule.stage_map(d) for d in schedule.directions]
    counts = [len(p.halfblocks) for p in stage_partition(cfg, S)]
    unit = 1e6

    def score(c):
        cost = [Fraction(round(x / unit)) for x in stage_costs(cfg, c)]
        dur = lambda t: cost[t.stage] * (1 if t.kind.value == "F" else 2)  # noqa: E731
        starts = list_schedule(schedule.per_device, schedule.dependencies, dur)
        mk = max(st + dur(t) for t, st in starts.items())
        ld = device_loads(cfg, c, maps)
        return (mk, max(ld), sum(x * x for x in ld))

    best = score(counts)
    improved = True
    while improved:
        improved = False
        for b in range(S - 1):
            for delta in (1, -1):  # one half-block from stage b to b+1, or back
                c = list(counts)
                c[b] -= delta
                c[b + 1] += delta
                if min(c) < 0:
                    continue
                sc = score(c)
                if sc < best:
                    best, counts, improved = sc, c, True
    return counts


# -- measured-cost partitioner ------------------------------------------------
# Task kinds of the as-executed replay (schedule.analysis.replay_times): F,
# B (= backward with its micro-batch's weight gradients, the paper's model),
# Bd (= the input-gradient chain the step runs when weight gradients are
# deferred) and W (= one stage replica's deferred weight-gradient GEMMs over
# its n_rep micro-batches).  A stage's time of each kind is modelled as
# linear in its content: attention half-blocks, MLP half-blocks, the LM head
# (+ final LN + cross-entropy) and the embedding.
COST_TERMS = ("attn", "mlp", "head", "embed")
COST_KINDS = ("F", "B", "Bd", "W")


def _stage_terms(counts) -> list:
    out, start = [], 0
    S = len(counts)
    for s, c in enumerate(counts):
        n_attn = sum(1 for hb in range(start, start + c) if hb % 2 == 0)
        out.append((n_attn, c - n_attn, 1 if s == S - 1 else 0, 1 if s == 0 else 0))
        start += c
    return out


def fit_task_costs(counts, times: dict, n_rep: int, *more) -> dict:
    """Least-squares fit of ``{kind: {term: ms}}`` (COST_KINDS x COST_TERMS)
    to measured task times ``{(direction, stage, kind): ms}``
    (``Trainer.measure_task_times``) of a run with partition ``counts``
    (every direction's replica of a stage is one sample; further runs as
    ``(counts, times, n_rep)`` triples in ``more``).  W is stored per
    micro-batch (the measured block covers the replica's ``n_rep``)."""
    rows, ys = [], {k: [] for k in COST_KINDS}
    for cnt, tm, nr in ((counts, times, n_rep),) + tuple(more):
        terms = _stage_terms(cnt)
        for dr, s, _k in sorted(k for k in tm if k[2] == "F"):
            rows.append(terms[s])
            for kind in COST_KINDS:
                ys[kind].append(tm[(dr, s, kind)] / (nr if kind == "W" else 1))
    X = torch.tensor(rows, dtype=torch.float64)
    out = {}
    for kind in COST_KINDS:
        y = torch.tensor(ys[kind], dtype=torch.float64)[:, None]
        c = torch.linalg.lstsq(X, y).solution[:, 0]
        out[kind] = {t: max(0.0, float(v)) for t, v in zip(COST_TERMS, c)}
    return out


def modelled_task_times(counts, costs: dict, schedule) -> dict:
    """Task times ``{(direction, stage, kind): ms}`` of partition ``counts``
    under the linear cost table ``costs`` (``fit_task_costs``; W scaled to
    the schedule's micro-batches per replica)."""
    out = {}
    n_rep = schedule.N // len(schedule.directions)
    for s, tm in enumerate(_stage_terms(counts)):
        for kind in COST_KINDS:
            v = sum(n * costs[kind][t] for n, t in zip(tm, COST_TERMS)) * (n_rep if kind == "W" else 1)
            for dr in schedule.directions:
                out[(dr, s, kind)] = v
    return out


def calibrated_counts(cfg: ModelConfig, schedule, costs: dict, *, deferred_w: bool = True, start=None) -> list[int]:
    """Half-blocks per stage minimising the replayed makespan of
    ``schedule``'s fixed per-device orders (reference ``list_schedule``,
    fusion.py:34-77, one GPU per logical device, free communication) under
    the MEASURED cost table ``costs`` -- as the step executes it
    (``deferred_w``: weight gradients deferred into one block per stage
    replica after its last backward; else the paper's B = F + W model).
    Local search from ``start`` (default :func:`balanced_counts`): move one
    half-block between any two stages while the makespan (then the most
    loaded device) improves; every stage but the LM-head stage keeps at least
    one half-block (no pure pass-through hops).  Deterministic."""
    from .schedule.analysis import replay_times

    S = schedule.num_stages
    counts = list(start) if start is not None else balanced_counts(cfg, schedule)

    def score(c):
        r = replay_times(schedule, modelled_task_times(c, costs, schedule), deferred_w)
        return (round(r["makespan_ms"], 6), round(max(r["busy_ms_per_device"]), 6))

    best = score(counts)
    improved = True
    while improved:
        improved = False
        for b in range(S):
            for j in range(S):
                if j == b or counts[b] <= (0 if b == S - 1 else 1):
                    continue
                c = list(counts)
                c[b] -= 1
                c[j] += 1
                sc = score(c)
                if sc < best:
                    best, counts, improved = sc, c, True
    return counts


def load_calibration(name: str):
    """The committed B200 cost table of config ``name``
    (``paper_2410_19367_b200/calibration/<name>.json``: ``costs`` as fitted
    by :func:`fit_task_costs` from a bench run's measured task times, with
    provenance), or None."""
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "calibration", f"{name}.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f)["costs"]


def resolve_partition(cfg: ModelConfig, schedule, partition="balanced") -> list[int]:
    """Half-blocks per stage for ``partition``: "uniform" (stage_partition's
    rule), "balanced" (FLOP cost model, :func:`balanced_counts`),
    "calibrated" (measured B200 cost table of the config,
    :func:`calibrated_counts`; ValueError when the config has none), "auto"
    (calibrated when a table exists, else balanced) or explicit counts."""
    if isinstance(partition, str):
        if partition == "auto":
            partition = "calibrated" if load_calibration(cfg.name) is not None else "balanced"
        if partition == "uniform":
            return [len(p.halfblocks) for p in stage_partition(cfg, schedule.num_stages)]
        if partition == "balanced":
            return balanced_counts(cfg, schedule)
        if partition == "calibrated":
            costs = load_calibration(cfg.name)
            if costs is None:
                raise ValueError(f"no B200 cost calibration for config {cfg.name!r} "
                                 f"(tools/calibrate.py writes calibration/<config>.json)")
            return calibrated_counts(cfg, schedule, costs)
        raise ValueError(f"unknown partition {partition!r}")
    return [int(c) for c in partition]


def param_specs(cfg: ModelConfig):
    """(name, shape, kind) for every parameter in a canonical order.
    kind: 'w' (N(0,.02)), 'wo' (scaled output proj), 'b' (zero), 'g' (one)."""
    h, f, V, S = cfg.hidden, cfg.ffn, cfg.vocab, cfg.seq
    out = [("embed.wte", (V, h), "w"), ("embed.wpe", (S, h), "w")]
    for l in range(cfg.layers):
        p = f"layers.{l}."
        out += [(p + "ln1.w", (h,), "g"), (p + "ln1.b", (h,), "b"),
                (p + "attn.qkv.w", (3 * h, h), "w"), (p + "attn.qkv.b", (3 * h,), "b"),
                (p + "attn.proj.w", (h, h), "wo"), (p + "attn.proj.b", (h,), "b"),
                (p + "ln2.w", (h,), "g"), (p + "ln2.b", (h,), "b"),
                (p + "mlp.fc1.w", (f, h), "w"), (p + "mlp.fc1.b", (f,), "b"),
                (p + "mlp.fc2.w", (h, f), "wo"), (p + "mlp.fc2.b", (h,), "b")]
    out += [("head.lnf.w", (h,), "g"), ("head.lnf.b", (h,), "b"), ("head.lm.w", (V, h), "w")]
    return out


def halfblock_param_names(hb: int) -> list[str]:
    l, half = divmod(hb, 2)
    p = f"layers.{l}."
    if half == 0:
        return [p + "ln1.w", p + "ln1.b", p + "attn.qkv.w", p + "attn.qkv.b", p + "attn.proj.w", p + "attn.proj.b"]
    return [p + "ln2.w", p + "ln2.b", p + "mlp.fc1.w", p + "mlp.fc1.b", p + "mlp.fc2.w", p + "mlp.fc2.b"]


def stage_param_names(plan: StagePlan) -> list[str]:
    names = ["embed.wte", "embed.wpe"] if plan.embed else []
    for hb in plan.halfblocks:
        names += halfblock_param_names(hb)
    if plan.head:
        names += ["head.lnf.w", "head.lnf.b", "head.lm.w"]
    return names


def init_params(cfg: ModelConfig, seed: int = 1234, *, device="cpu", dtype=torch.float32,
                perturb: bool = False) -> dict:
    """Seeded initial parameters {name: tensor}; identical for every replica."""
    gen = torch.Generator(device=device).manual_seed(seed)
    out = {}
    std = 0.02
    std_o = 0.02 / math.sqrt(2 * cfg.layers)
    for name, shape, kind in param_specs(cfg):
        if kind in ("w", "wo"):
            t = torch.randn(shape, generator=gen, device=device, dtype=torch.float32) * (std if kind == "w" else std_o)
        elif kind == "b":
            t = torch.zeros(shape, device=device, dtype=torch.float32)
            if perturb:
                t += 0.02 * torch.randn(shape, generator=gen, device=device, dtype=torch.float32)
        else:
            t = torch.ones(shape, device=device, dtype=torch.float32)
            if perturb:
                t += 0.05 * torch.randn(shape, generator=gen, device=device, dtype=torch.float32)
        out[name] = t.to(dtype)
    return out


@dataclass
class OptimConfig:
    """AdamW hyper-parameters of the single post-flush update."""
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.0


def synthetic_batch(cfg: ModelConfig, N: int, seed: int = 1234):
    """i.i.d. uniform token ids [N, B, S] and targets (GPT: ids shifted by
    one; BERT: independent random targets), from a seeded CPU generator
    (SURVEY §8(d))."""
    gen = torch.Generator().manual_seed(seed)
    toks = torch.randint(0, cfg.vocab, (N, cfg.micro_batch, cfg.seq + 1), generator=gen, dtype=torch.int64)
    if cfg.causal:
        return toks[..., :-1].contiguous(), toks[..., 1:].contiguous()
    tgt = torch.randint(0, cfg.vocab, (N, cfg.micro_batch, cfg.seq), generator=gen, dtype=torch.int64)
    return toks[..., :-1].contiguous(), tgt
