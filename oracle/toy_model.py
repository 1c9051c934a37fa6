"""TEST INFRASTRUCTURE ONLY -- the SPEC's ToyModel runtime (fp64, SGD).

Restates the reference SPEC ``runtime`` module literally:

  * ``ToyModel``: one dense weight matrix per stage
    (``stage_dims`` = layer widths, stage s maps width dims[s] -> dims[s+1]),
    optional elementwise activation between stages, mean-squared-error over
    the final output;
  * ``run_schedule_numeric(schedule, model, batch, seed)``:
    the reference per-device orders executed with message passing -- the
    SAME executor the GPT oracle uses (``gpt_oracle.execute_orders``), so
    the known answers below pin that executor;
  * ``sequential_baseline``: one worker, N micro-batches,
    mean loss, one update;
  * plain SGD with a fixed learning rate, replica gradients
    averaged, one update after the flush.

Its known answers (tests/test_oracle_pinning.py): the
identity-initialised 1F1B D=2 N=2 closed-form loss, the N=1 scalar MSE
derivative, linearity of accumulation (N=4 == mean of 4 single-micro-batch
gradients) and schedule independence within 1e-9 (fp64).
"""
from __future__ import annotations

import json
from dataclasses import dataclass

import torch

from .gpt_oracle import execute_orders, replica_mean_grads

__all__ = ["ToyModel", "ToyStepResult", "toy_run_schedule_numeric", "toy_sequential_baseline"]


@dataclass
class ToyModel:
    stage_params: list          # [num_stages] fp64 weight matrices, stage s: [dims[s], dims[s+1]]
    stage_dims: list            # layer widths, len = num_stages + 1
    activation: str = "none"    # "none" | "tanh" (applied after every stage but the last)
    lr: float = 0.1

    @staticmethod
    def random(stage_dims, seed: int = 0, activation: str = "none", lr: float = 0.1) -> "ToyModel":
        g = torch.Generator().manual_seed(seed)
        ws = [torch.randn(a, b, generator=g, dtype=torch.float64) / a ** 0.5
              for a, b in zip(stage_dims[:-1], stage_dims[1:])]
        return ToyModel(ws, list(stage_dims), activation, lr)

    @staticmethod
    def identity(num_stages: int, width: int = 1, lr: float = 0.1) -> "ToyModel":
        eye = torch.eye(width, dtype=torch.float64)
        return ToyModel([eye.clone() for _ in range(num_stages)], [width] * (num_stages + 1), "none", lr)

    @property
    def num_stages(self) -> int:
        return len(self.stage_params)


@dataclass
class ToyStepResult:
    grads: list      # per-stage gradient (replica mean), fp64
    weights: list    # per-stage weights after the single SGD update
    loss: float      # mean over the N micro-batches
    losses: torch.Tensor


def _stage(model: ToyModel, W, s, x):
    y = x @ W
    if model.activation == "tanh" and s < model.num_stages - 1:
        y = torch.tanh(y)
    return y


def _mse(y, t):
    return ((y - t) ** 2).mean()


def _sgd(model: ToyModel, grads):
    return [w - model.lr * g for w, g in zip(model.stage_params, grads)]


def toy_sequential_baseline(model: ToyModel, batch, seed: int = 0) -> ToyStepResult:
    """single worker, mean over N micro-batches, one update.
    ``batch`` = (inputs [N, B, dims[0]], targets [N, B, dims[-1]]); ``seed``
    is accepted for the SPEC signature (the step is deterministic)."""
    xs, ts = batch
    N = xs.shape[0]
    W = [w.detach().clone().requires_grad_(True) for w in model.stage_params]
    losses = torch.zeros(N, dtype=torch.float64)
    for i in range(N):
        y = xs[i]
        for s, w in enumerate(W):
            y = _stage(model, w, s, y)
        loss = _mse(y, ts[i])
        (loss / N).backward()
        losses[i] = loss.detach()
    grads = [w.grad.detach().clone() for w in W]
    return ToyStepResult(grads, _sgd(model, grads), losses.mean().item(), losses)


def toy_run_schedule_numeric(schedule_json, model: ToyModel, batch, seed: int = 0) -> ToyStepResult:
    """SPEC.md:426-434 on the ToyModel: the schedule's total stage count must
    equal the model's; bidirectional schedules instantiate two
    identically initialised replicas whose gradients are averaged before
    the single SGD update."""
    sch = json.loads(schedule_json) if isinstance(schedule_json, str) else schedule_json
    S_tot = sch["D"] * sch["v"]
    if S_tot != model.num_stages:
        raise ValueError(f"ShapeMismatch: schedule has {S_tot} stages, model {model.num_stages}")
    xs, ts = batch
    N = xs.shape[0]
    if N != sch["N"]:
        raise ValueError(f"ShapeMismatch: batch has {N} micro-batches, schedule {sch['N']}")
    dirs = [m["direction"] for m in sch["stage_maps"]]
    names = [f"w{s}" for s in range(S_tot)]
    replicas = {d: {n: w.detach().clone().requires_grad_(True) for n, w in zip(names, model.stage_params)}
                for d in dirs}
    last = S_tot - 1

    def stage_fn(P, s, x_in, mb):
        x = xs[mb - 1] if s == 0 else x_in
        y = _stage(model, P[names[s]], s, x)
        return _mse(y, ts[mb - 1]) if s == last else y

    losses = execute_orders(sch, replicas, stage_fn, N)
    g = replica_mean_grads(replicas, names)
    grads = [g[n] for n in names]
    return ToyStepResult(grads, _sgd(model, grads), losses.mean().item(), losses)
