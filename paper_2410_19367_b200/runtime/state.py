"""Per-stage parameter / gradient / optimizer storage and the buffer pool.

HBM layout: every (direction replica, virtual stage) owns one
flat parameter buffer in the compute dtype plus one flat fp32 gradient
buffer with identical offsets (64-element aligned, so every tensor view is
16-byte aligned for the vectorised kernels and TMA).  The AdamW master
weights and moments are flat fp32 buffers owned by the process that runs
that stage's update.  Flat buffers make the eager replica-pair gradient
sync one contiguous collective (or one fused kernel) per stage.
"""
from __future__ import annotations

import math
from collections import defaultdict

import torch

from ..model import ModelConfig, StagePlan, param_specs, stage_param_names

__all__ = ["StageParams", "BufferPool", "ALIGN"]

ALIGN = 64


GEMM_WEIGHTS = ("attn.qkv.w", "attn.proj.w", "mlp.fc1.w", "mlp.fc2.w", "head.lm.w")


class StageParams:
    """Flat storage of one stage replica's parameters and gradients."""

    def __init__(self, cfg: ModelConfig, plan: StagePlan, dtype: torch.dtype, device, share_params=None):
        """``share_params``: another replica's StageParams of the same stage
        whose working weights this replica uses (co-resident replicas are
        bit-identical at every step; gradients stay separate)."""
        shapes = {n: s for n, s, _ in param_specs(cfg)}
        # GEMM-written weight gradients last: the first backward of an
        # iteration writes them (beta = 0) instead of accumulating, so only the
        # leading atomically-accumulated part (embeddings, biases, LayerNorm)
        # needs zeroing before the iteration (``zero_numel``)
        names = stage_param_names(plan)
        self.names = ([n for n in names if not n.endswith(GEMM_WEIGHTS)] +
                      [n for n in names if n.endswith(GEMM_WEIGHTS)])
        self.offsets = {}
        off = 0
        self.zero_numel = None
        for n in self.names:
            if self.zero_numel is None and n.endswith(GEMM_WEIGHTS):
                self.zero_numel = off
            self.offsets[n] = off
            off += -(-math.prod(shapes[n]) // ALIGN) * ALIGN
        self.numel = max(off, ALIGN)
        if self.zero_numel is None:
            self.zero_numel = self.numel
        self.dtype = dtype
        self.device = torch.device(device)
        self.flat = share_params.flat if share_params is not None else torch.zeros(self.numel, dtype=dtype,
                                                                                    device=device)
        self.grad = torch.zeros(self.numel, dtype=torch.float32, device=device)
        self.shapes = {n: tuple(shapes[n]) for n in self.names}
        self.p = {n: self._view(self.flat, n) for n in self.names}
        self.g = {n: self._view(self.grad, n) for n in self.names}
        self.master = self.m = self.v = None

    def _view(self, flat, n):
        o = self.offsets[n]
        return flat[o:o + math.prod(self.shapes[n])].view(self.shapes[n])

    def load(self, params: dict) -> None:
        for n in self.names:
            self.p[n].copy_(params[n].to(device=self.device, dtype=self.dtype))

    def init_optimizer(self, params: dict | None = None) -> None:
        """Allocate fp32 master/m/v; master from ``params`` (exact fp32) when
        given, else from the working copy."""
        self.master = torch.zeros(self.numel, dtype=torch.float32, device=self.device)
        self.m = torch.zeros_like(self.master)
        self.v = torch.zeros_like(self.master)
        for n in self.names:
            o = self.offsets[n]
            src = params[n] if params is not None else self.p[n]
            self.master[o:o + src.numel()].copy_(src.reshape(-1).to(device=self.device, dtype=torch.float32))

    def master_view(self, n):
        return self._view(self.master, n)


class BufferPool:
    """Event-guarded free lists of device buffers keyed by (shape, dtype).

    ``get`` hands out a free buffer after making the requesting stream wait
    for the event recorded when it was released (so reuse across the
    per-logical-device streams is ordered); ``put_all`` releases a batch of
    buffers under one event.  After the first iteration every request is a
    hit, so the steady state allocates nothing.
    """

    def __init__(self, device):
        self.device = torch.device(device)
        self.free = defaultdict(list)
        self.allocated_bytes = 0
        self.foreign: set = set()   # data_ptr()s of buffers the pool must never take (transport slots)

    def get(self, shape, dtype, stream):
        """A free buffer of this shape, preferring one released on ``stream``
        itself (stream order already covers its last use, no cross-stream
        dependency); otherwise the most recently released one, after making
        ``stream`` wait for its release event."""
        key = (tuple(shape), dtype)
        lst = self.free[key]
        if lst:
            sid = stream.cuda_stream
            for i in range(len(lst) - 1, -1, -1):
                if lst[i][2] == sid:
                    return lst.pop(i)[0]
            t, ev, _ = lst.pop()
            if ev is not None:
                stream.wait_event(ev)
            return t
        with torch.cuda.stream(stream):
            t = torch.empty(key[0], dtype=dtype, device=self.device)
        self.allocated_bytes += t.numel() * t.element_size()
        return t

    def put_all(self, tensors, event, stream=None) -> None:
        """Release ``tensors`` once ``event`` (recorded on ``stream``) fires."""
        sid = stream.cuda_stream if stream is not None else None
        for t in tensors:
            if t is not None and t.data_ptr() not in self.foreign:
                self.free[(tuple(t.shape), t.dtype)].append((t, event, sid))

    def forget_events(self) -> None:
        """Drop the release events of every free buffer (call only when the
        device is idle, e.g. after capturing a CUDA graph whose events must
        not be waited on outside it)."""
        for lst in self.free.values():
            for i, (t, _ev, sid) in enumerate(lst):
                lst[i] = (t, None, sid)
