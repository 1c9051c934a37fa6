"""The SPEC-shaped train-step entry: ``train_step(schedule, model, batch, seed)``.

The reference specifies (but does not implement) the runtime entry
``run_schedule_numeric(schedule, model, batch, seed) -> StepResult`` with
per-stage gradients, the weights after the single post-flush update and the
loss.  This module is that call on the B200: it builds (or
reuses) a :class:`~.executor.Trainer` for the schedule / model, runs ONE
iteration -- every per-device list in the bit-exact reference order, eager
replica-pair gradient sync, one AdamW update -- and returns the results as
host tensors.

For throughput use the :class:`Trainer` directly (``Trainer.train_step``
keeps everything on the device and returns only the loss vector); this
entry synchronises and copies gradients / parameters to the host.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from ..model import CONFIGS, ModelConfig, OptimConfig, init_params
from ..schedule import Schedule, load_schedule
from .executor import Trainer

__all__ = ["StepResult", "train_step", "run_schedule_numeric"]


@dataclass
class StepResult:
    """SPEC.md:419-424 ``StepResult``: per-micro-batch losses (index =
    micro-batch id - 1) and their mean; the replica-mean gradients the
    update applied (pre-update, fp32); the updated parameters (fp32 master
    weights); the Trainer, for further steps."""
    losses: torch.Tensor
    loss: float
    grads: dict
    params: dict
    trainer: Trainer


def train_step(schedule: Schedule | str, model: ModelConfig | str, batch, seed: int = 1234, *,
               dtype=torch.bfloat16, optim: OptimConfig | None = None, params: dict | None = None,
               partition="uniform", trainer: Trainer | None = None, dist_ctx=None, device=None) -> StepResult:
    """One BitPipe iteration of ``schedule`` on ``model`` over ``batch``.

    schedule -- a :class:`Schedule` or its JSON wire format (``dump_schedule``,
                reference schedules.py:301-356);
    model    -- a :class:`ModelConfig` or a name in ``CONFIGS``;
    batch    -- (tokens, targets), integer tensors [N, B, S] (host or device);
    seed     -- parameter initialisation seed (ignored when ``params`` or
                ``trainer`` is given); both replicas start identical.

    Pass ``trainer=result.trainer`` to continue from a previous step (same
    schedule and model).  Raises ``ValueError`` when the batch does not
    have the schedule's N micro-batches (SPEC ShapeMismatch) and
    ``RuntimeError`` without a CUDA device (there is no CPU fallback).
    """
    if isinstance(schedule, str):
        schedule = load_schedule(schedule)
    cfg = CONFIGS[model] if isinstance(model, str) else model
    tokens, targets = batch
    want = (schedule.N, cfg.micro_batch, cfg.seq)
    if tuple(tokens.shape) != want or tuple(targets.shape) != want:
        raise ValueError(f"ShapeMismatch: batch {tuple(tokens.shape)} / {tuple(targets.shape)}, "
                         f"schedule x model need {want}")
    if trainer is None:
        if params is None:
            params = init_params(cfg, seed)
        trainer = Trainer(cfg, schedule, dtype=dtype, optim=optim, params=params, partition=partition,
                          dist_ctx=dist_ctx, device=device)
    elif trainer.sched is not schedule and trainer.sched != schedule:
        raise ValueError("trainer was built for a different schedule")
    dev = trainer.device
    out = trainer.train_step(tokens.to(dev, torch.int32, non_blocking=True),
                             targets.to(dev, torch.int32, non_blocking=True))
    losses = out.losses.detach().double().cpu()
    if dist_ctx is None:
        grads = trainer.mean_grads()
    else:  # this rank's stages; the pair mean was applied inside the update
        grads = trainer.gather("grads")
    params_after = trainer.gather("master")
    return StepResult(losses, losses.mean().item() if dist_ctx is None else float("nan"), grads, params_after,
                      trainer)


run_schedule_numeric = train_step
