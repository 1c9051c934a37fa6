"""The BitPipe train step: executes a :class:`Schedule` on CUDA streams.

This is the B200 realisation of the reference SPEC's absent ``runtime``
module (``run_schedule_numeric``) for the transformer model
of :mod:`..model`:

* every logical device ``d`` of the schedule gets its own CUDA stream and
  runs ``schedule.per_device[d]`` strictly in list order (the order is the
  bit-exact reference order);
* activation / gradient messages are tag-addressed by (kind, direction,
  micro-batch, destination stage) -- never by arrival order -- because the
  reference orders are not FIFO-consistent per link;
* eager gradient synchronisation: as soon as a stage's last backward on a
  device is issued, that stage's replica-pair gradient mean and AdamW update
  are issued on the optimizer stream, overlapping the rest of the drain
  (PAPER.md:151-153);
* one weight update per iteration, after all uses of the stage's weights.

Placement modes
  coresident  (one process, one GPU): all D logical devices share the GPU,
              each on its own stream; messages are zero-copy hand-offs gated
              by CUDA events; the replica-pair "allreduce" is the fused
              (g_down + g_up)/2 read inside the Adam kernel.
  distributed (one process per GPU, world == D, rank == logical device):
              messages move over NCCL P2P (torch.distributed) with receives
              posted up-front in the sender's order on one group per link
              direction; the pair mean is a 2-rank NCCL all-reduce on a
              per-(pair, stage) group, followed by the local Adam.
"""
from __future__ import annotations

import os
import time
from dataclasses import dataclass

import torch

from ..model import ModelConfig, OptimConfig, resolve_partition, stage_partition
from ..schedule import Direction, Schedule, TaskKind, canonical_replay
from ..schedule.analysis import WeightGradTask, replay_times
from . import ops
from .lib import OPT_GEMM_PICK
from .compute import StageCompute
from .state import GEMM_WEIGHTS, BufferPool, StageParams

__all__ = ["Trainer", "StepOutput", "issue_order", "drive", "choose_deferred_stages", "replay_times",
           "WeightGradTask"]


@dataclass
class StepOutput:
    losses: torch.Tensor           # [N] fp32 device tensor, index = micro-batch id - 1
    step: int
    task_events: dict | None = None


def issue_order(schedule: Schedule):
    """A single-thread issue order over all (device, position) pairs that is a
    topological order of dataflow + per-device order: sort by the canonical
    ASAP start time (dependencies end no later than a task starts and have
    positive duration), ties by device then position."""
    starts, _ = canonical_replay(schedule)
    items = []
    for d, row in enumerate(schedule.per_device):
        for i, t in enumerate(row):
            items.append((starts[t], d, i, t))
    items.sort(key=lambda x: (x[0], x[1], x[2]))
    return [(d, i, t) for _, d, i, t in items]


def choose_deferred_stages(slot_bytes: dict, work: dict, budget: float) -> set:
    """Stages whose weight gradients are deferred: all of them when their
    slots fit ``budget`` bytes, else greedily the stages with the most
    weight-GEMM work per slot byte (ties: lower stage first) while they fit;
    the rest keep per-micro-batch weight gradients.  So a model too large for
    every slot (e.g. the GPT-10B width) still defers most of its GEMMs."""
    if sum(slot_bytes.values()) <= budget:
        return set(slot_bytes)
    chosen, used = set(), 0
    for s in sorted(slot_bytes, key=lambda s: (-work[s] / max(1, slot_bytes[s]), s)):
        if slot_bytes[s] and used + slot_bytes[s] <= budget:
            chosen.add(s)
            used += slot_bytes[s]
    return chosen


def drive(order, num_stages, last_b, *, forward, backward, send, recv, stage_done, dev_of, stashes=None):
    """Issue every task of ``order`` (list of (device, position, Task)).

    Pure host-side control flow shared by the CUDA executor and the
    multi-process CPU tests: forward(d, t, x0) -> (stash, out|None);
    backward(d, t, stash, dy) -> (dx|None, event); send/recv move
    tag-addressed messages keyed (kind, direction, mb, destination stage);
    stage_done(direction, stage, d, event) fires after the LAST backward of
    that (direction, stage) on device d -- the eager sync launch point.
    Returns the leftover (msgs, stashes), both empty for a valid schedule.
    ``stashes`` (optional) is the live dict of forward stashes keyed
    (direction, micro-batch, stage), readable from the callbacks.
    """
    msgs: dict = {}
    stashes = {} if stashes is None else stashes
    last = num_stages - 1
    for d, i, t in order:
        dr, s, mb = t.direction, t.stage, t.micro_batch
        if t.kind is TaskKind.FORWARD:
            x0 = recv(msgs, ("act", dr, mb, s), d) if s > 0 else None
            stash, out = forward(d, t, x0)
            stashes[(dr, mb, s)] = stash
            if out is not None:
                send(msgs, ("act", dr, mb, s + 1), out, d, dev_of(dr, s + 1))
        else:
            dy = recv(msgs, ("grad", dr, mb, s), d) if s < last else None
            stash = stashes.pop((dr, mb, s))
            dx, ev = backward(d, t, stash, dy)
            msg_ev, done_ev = ev if isinstance(ev, tuple) else (ev, ev)
            if dx is not None:
                send(msgs, ("grad", dr, mb, s - 1), dx, d, dev_of(dr, s - 1), event=msg_ev)
            if last_b[d].get((dr, s)) == i:
                stage_done(dr, s, d, done_ev)
    return msgs, stashes


class Trainer:
    """Executes BitPipe (or any schedule from :mod:`..schedule`) on one GPU
    (coresident) or one process per logical device (distributed).

    ``train_step(tokens, targets)`` runs one iteration: N micro-batches
    through the schedule, eager replica-pair gradient sync, one AdamW update.
    """

    def __init__(self, cfg: ModelConfig, schedule: Schedule, *, dtype=torch.bfloat16, optim: OptimConfig | None = None,
                 params: dict | None = None, seed: int = 1234, device=None, dist_ctx=None, record_timeline=False,
                 serial_streams: bool = False, partition="uniform", stream_priority=None, wgrad_stream=None,
                 defer_wgrad=None, eager_sync=None):
        if not torch.cuda.is_available():
            raise RuntimeError("BitPipe Trainer needs a CUDA device (no CPU fallback)")
        ops.lib()  # fail loudly now if the kernel library is missing
        self.cfg, self.sched = cfg, schedule
        self.dtype = dtype
        self.optim = optim or OptimConfig()
        self.D, self.v = schedule.D, schedule.v
        self.S = schedule.num_stages
        self.N = schedule.N
        self.dirs = list(schedule.directions)
        self.bidir = len(self.dirs) == 2
        self.n_rep = self.N // len(self.dirs)
        # layer -> stage partition: "uniform", "balanced" (FLOP-cost-balanced
        # for this schedule), "calibrated" (measured B200 cost table, replayed
        # as executed), "auto" or explicit half-blocks per stage
        # (model.resolve_partition)
        counts = resolve_partition(cfg, schedule, partition)
        self.plans = stage_partition(cfg, self.S, counts)
        self.partition = [len(p.halfblocks) for p in self.plans]
        self.dist = dist_ctx
        self.device = torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")
        torch.cuda.set_device(self.device)
        self.local_devices = list(range(self.D)) if dist_ctx is None else [dist_ctx.dev]
        self.record_timeline = record_timeline
        self.step_count = 0
        # eager gradient synchronisation: a
        # stage's replica-pair sync + update is issued right after its last
        # backward on the device; False = "BitPipe w/o E":
        # every sync waits for the device's whole task list
        if eager_sync is None:
            import os
            eager_sync = os.environ.get("BP_EAGER_SYNC", "1") == "1"
        self.eager_sync = bool(eager_sync)

        # -- parameters: one StageParams per (direction, stage) held locally --
        if params is None:
            from ..model import init_params
            params = init_params(cfg, seed, device=self.device)
        self.stage_params: dict = {}
        self.compute: dict = {}
        grad_scale = 1.0 / self.n_rep
        if defer_wgrad is None:  # env BP_DEFER_WGRAD=0/1 forces; default: per stage, while the slots fit
            import os
            env = os.environ.get("BP_DEFER_WGRAD")
            if env is not None:
                defer_wgrad = env == "1"
            else:
                defer_wgrad = self._deferred_stages(dtype, 0.4 * torch.cuda.get_device_properties(
                    self.device).total_memory)
        # per-stage decision: a set of stages, or all / none
        defer_of = (lambda s: s in defer_wgrad) if isinstance(defer_wgrad, (set, frozenset)) else \
            (lambda s, v=bool(defer_wgrad): v)
        self.deferred_stages = sorted(s for s in range(self.S) if defer_of(s))
        for dr in self.dirs:
            smap = schedule.stage_map(dr)
            for s in range(self.S):
                if smap.device_of(s) not in self.local_devices:
                    continue
                # co-resident: the second direction's replica reads the first's
                # working weights (bit-identical by construction);
                # AdamW then writes one bf16 copy per stage
                other = self.stage_params.get((self.dirs[0], s)) if dist_ctx is None and dr != self.dirs[0] else None
                sp = StageParams(cfg, self.plans[s], dtype, self.device, share_params=other)
                if other is None:
                    sp.load(params)
                self.stage_params[(dr, s)] = sp
                self.compute[(dr, s)] = StageCompute(cfg, self.plans[s], sp, grad_scale=grad_scale, n_rep=self.n_rep,
                                                     defer_wgrad=defer_of(s))
        # co-resident bidirectional: one deferred weight-gradient GEMM per
        # weight over both replicas' micro-batches (shared slots, K = N M),
        # issued on the optimizer stream when both replicas are done
        self.combined_stages = (set(self.deferred_stages) if dist_ctx is None and self.bidir and self.n_rep > 1
                                else set())
        self.combined_wgrad = bool(self.combined_stages)
        if self.combined_wgrad:
            for s in sorted(self.combined_stages):
                c0, c1 = self.compute[(self.dirs[0], s)], self.compute[(self.dirs[1], s)]
                c1._slots = c0._slots
                c0.slot_total = c1.slot_total = 2 * self.n_rep
                c1.slot_base = self.n_rep
                c0.combined_wgrad = c1.combined_wgrad = True
        if dist_ctx is None:  # all stages local: fuse each stage's last output-bias gradient
            for dr in self.dirs:  # into the next stage's message-producing LayerNorm backward
                for s in range(1, self.S):
                    prev, cur = self.compute[(dr, s - 1)], self.compute[(dr, s)]
                    if prev.plan.halfblocks and (cur.plan.halfblocks or cur.plan.head):
                        cur.prev_out_bias = prev._out_bias_grad(len(prev.plan.halfblocks) - 1)
                        prev.out_bias_by_next = True
        # optimizer state: one master/m/v per stage present locally (coresident:
        # shared by the two replicas; distributed: per local replica)
        self.opt_owner: dict = {}
        for (dr, s), sp in self.stage_params.items():
            key = s if dist_ctx is None else (dr, s)
            if key not in self.opt_owner:
                sp.init_optimizer(params)
                self.opt_owner[key] = sp
        del params

        # -- streams, pools, workspaces ------------------------------------------------
        if serial_streams:   # all logical devices on one stream (no cross-device kernel concurrency)
            one = torch.cuda.Stream(device=self.device)
            self.streams = {d: one for d in self.local_devices}
        else:
            prio = self._stream_priorities(stream_priority)
            self.streams = {d: torch.cuda.Stream(device=self.device, priority=prio.get(d, 0))
                            for d in self.local_devices}
        self.opt_stream = torch.cuda.Stream(device=self.device)
        # co-resident: per-stage optimizer work (combined weight-gradient GEMMs
        # + AdamW) round-robin over BP_OPT_STREAMS streams so the stages that
        # finish together in the drain overlap (1 = one serial stream)
        import os
        nopt = max(1, int(os.environ.get("BP_OPT_STREAMS", "1")))
        if len(self.local_devices) > 1 and not serial_streams and os.environ.get("BP_GEMM_PICK", "") == "":
            # several logical devices' streams share this GPU: pick GEMM tiles
            # for per-tile efficiency (csrc/gemm.cu pick_tc2_bn, BP_OPT_GEMM_PICK;
            # BP_GEMM_PICK=0 keeps the wave-quantisation model)
            ops.set_option(OPT_GEMM_PICK, 1)
        self.opt_streams = [self.opt_stream] + [torch.cuda.Stream(device=self.device) for _ in range(nopt - 1)]
        # distributed: one optimizer stream per local stage -- each stage's
        # replica-pair sync (NCCL all-reduce or peer-read AdamW) must not be
        # ordered behind another stage's, whose partner may reach it later
        # (distributed.sync_order_acyclic)
        self.stage_streams: dict = {}
        if dist_ctx is not None:
            for (_dr, s) in self.stage_params:
                if s not in self.stage_streams:
                    self.stage_streams[s] = torch.cuda.Stream(device=self.device)
                    self.opt_streams.append(self.stage_streams[s])
        # weight-gradient GEMMs on a side stream per logical device, off the
        # critical path of the backward chain (the message to the previous
        # stage no longer waits for them; +0.5 % co-resident, more concurrency
        # per GPU in distributed mode); env BP_WGRAD_STREAM=0 turns it off
        import os
        if wgrad_stream is None:
            wgrad_stream = os.environ.get("BP_WGRAD_STREAM", "1") == "1"
        self.wstreams = ({d: torch.cuda.Stream(device=self.device) for d in self.local_devices}
                         if wgrad_stream and not serial_streams else {})
        self.pool = BufferPool(self.device)
        wsn = ops.attn_workspace_numel(cfg.micro_batch, cfg.seq, cfg.heads, cfg.head_dim)
        self.ws = {d: torch.empty(wsn, dtype=torch.float32, device=self.device) for d in self.local_devices}
        self.losses = torch.zeros(self.N, dtype=torch.float32, device=self.device)
        self.last_b = schedule.last_backward_positions()
        if dist_ctx is None:
            self.order = issue_order(schedule)
        else:
            d = dist_ctx.dev
            self.order = [(d, i, t) for i, t in enumerate(schedule.per_device[d])]
            dist_ctx.setup(self)
        self.iter_done = None
        self.timeline = None
        self.step_dev = torch.zeros(1, dtype=torch.int32, device=self.device)  # AdamW step on the device
        self._graph_state = None
        self._graph = None

    # ----------------------------------------------------------------- helpers --
    def _slot_bytes(self, dtype, stage=None) -> int:
        """Device memory the deferred weight-gradient slots of this process's
        stage replicas take (of one stage, or all): per half-block n_rep
        micro-batches of (attention) a, o, dy, dqkv = 6h or (MLP) m, g, dy,
        du = 2h + 2 ffn columns, plus LN-f output and logits on the head
        stage."""
        cfg = self.cfg
        esz = torch.empty(0, dtype=dtype).element_size()
        rows = self.n_rep * cfg.micro_batch * cfg.seq
        total = 0
        for dr in self.dirs:
            smap = self.sched.stage_map(dr)
            for s in range(self.S):
                if smap.device_of(s) not in self.local_devices or (stage is not None and s != stage):
                    continue
                for hb in self.plans[s].halfblocks:
                    total += rows * (6 * cfg.hidden if hb % 2 == 0 else 2 * cfg.hidden + 2 * cfg.ffn) * esz
                if self.plans[s].head:
                    total += rows * (cfg.hidden + cfg.vocab) * esz
        return total

    def _deferred_stages(self, dtype, budget: float) -> set:
        """Stages whose weight gradients are deferred to one K = N M GEMM per
        weight (``choose_deferred_stages`` over this process's slot sizes)."""
        cfg = self.cfg

        def work(s):   # weight-gradient FLOPs per micro-batch token of stage s
            w = sum(8 * cfg.hidden ** 2 if hb % 2 == 0 else 2 * cfg.hidden * cfg.ffn for hb in self.plans[s].halfblocks)
            return w + (cfg.hidden * cfg.vocab if self.plans[s].head else 0)

        return choose_deferred_stages({s: self._slot_bytes(dtype, s) for s in range(self.S)},
                                      {s: work(s) for s in range(self.S)}, budget)

    def _stream_priorities(self, mode) -> dict:
        """Co-resident CUDA stream priorities (lower = more urgent).  'tail'
        (the default): the logical devices whose lists finish last in the
        canonical replay get the highest priority, so the pipeline drain (few
        streams with work left) is shorter -- BERT-large D=4 N=8 +1.5 %
        (316 k vs 311-312 k tok/s, same box), GPT-1.3B within noise; 'none'
        (argument or BP_STREAM_PRIORITY): all equal."""
        import os
        mode = mode or os.environ.get("BP_STREAM_PRIORITY") or "tail"
        if mode in (None, "", "none") or len(self.local_devices) < 2:
            return {}
        if mode != "tail":
            raise ValueError(f"unknown stream_priority {mode!r}")
        starts, _ = canonical_replay(self.sched)
        end = {d: max(starts[t] + self.sched.canonical_duration(t) for t in row)
               for d, row in enumerate(self.sched.per_device)}
        ranked = sorted(self.local_devices, key=lambda d: (-end[d], d))
        levels = sorted(set(end[d] for d in ranked), reverse=True)
        return {d: -max(0, 2 - levels.index(end[d])) for d in ranked}  # 3 levels: -2, -1, 0

    def stage_stream(self, s: int):
        """The optimizer stream of stage ``s`` (distributed mode)."""
        return self.stage_streams.get(s, self.opt_stream)

    def _dev_of(self, dr: Direction, s: int) -> int:
        return self.sched.stage_map(dr).device_of(s)

    def _zero_grads(self):
        """Zero the atomically accumulated gradients; the GEMM-written weight
        gradients are overwritten by each stage replica's first backward of
        the iteration (StageCompute.begin_iteration)."""
        for (dr, s), sp in self.stage_params.items():
            st = self.streams[self._dev_of(dr, s)]
            with torch.cuda.stream(st):
                sp.grad[:sp.zero_numel].zero_()
        for comp in self.compute.values():
            comp.begin_iteration()

    def _adam(self, stage_key, grads, params_out, stream, grad_scale=1.0, sl=None):
        owner = self.opt_owner[stage_key]
        o = self.optim
        a, b = sl if sl is not None else (0, owner.master.numel())
        ops.adam(owner.master[a:b], grads[0], grads[1] if len(grads) > 1 else None, owner.m[a:b], owner.v[a:b],
                 params_out[0], params_out[1] if len(params_out) > 1 else None,
                 lr=o.lr, beta1=o.beta1, beta2=o.beta2, eps=o.eps, weight_decay=o.weight_decay,
                 step=self.step_count, grad_scale=grad_scale, stream=stream, step_dev=self.step_dev)

    # ------------------------------------------------------------ CUDA graph --
    def enable_graph(self) -> None:
        """Replay the train step as one CUDA graph from the next call on
        (co-resident mode): the next ``train_step`` captures one iteration --
        every kernel, cross-stream event edge, eager AdamW -- and later calls
        copy the inputs into the captured buffers and replay it.  The step
        counter lives on the device (``bp_adam_dev``), the buffer pool is warm
        (no allocation inside the capture), so a replay is exactly one more
        eager iteration.  Call after at least one eager step."""
        if self.dist is not None:
            raise RuntimeError("CUDA-graph replay is for the co-resident executor (NCCL P2P is not captured)")
        if self.record_timeline:
            raise RuntimeError("disable record_timeline to capture the step")
        self._graph_state = "capture"

    def disable_graph(self) -> None:
        """Back to eager launches from the next ``train_step`` on (the
        captured graph is dropped; its buffers stay the pool's)."""
        if self._graph_state is None:
            return
        torch.cuda.synchronize(self.device)
        self._graph, self._graph_state = None, None
        self.iter_done = None
        self.pool.forget_events()

    def _graph_step(self, tokens, targets) -> StepOutput:
        if self._graph_state == "capture":
            self._g_tok = tokens.clone()
            self._g_tgt = targets.clone()
            torch.cuda.synchronize(self.device)
            self.pool.forget_events()  # the device is idle: no wait on events recorded outside the capture
            cap = torch.cuda.Stream(device=self.device)
            self.iter_done = None  # no edge to work outside the graph
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                self._step_body(self._g_tok, self._g_tgt)
            self._graph, self._graph_state = g, "replay"
            self.iter_done = None
            torch.cuda.synchronize(self.device)
            self.pool.forget_events()  # captured events must not be waited on outside the graph
        else:
            if tokens.data_ptr() != self._g_tok.data_ptr():
                self._g_tok.copy_(tokens, non_blocking=True)
                self._g_tgt.copy_(targets, non_blocking=True)
        self.step_count += 1
        self._graph.replay()
        return StepOutput(self.losses, self.step_count)

    # --------------------------------------------------------------- train step --
    def train_step(self, tokens: torch.Tensor, targets: torch.Tensor) -> StepOutput:
        """tokens/targets: int32 device tensors [N, B, S] already on this GPU."""
        if self._graph_state is not None:
            return self._graph_step(tokens, targets)
        self.step_count += 1
        return self._step_body(tokens, targets)

    def _step_body(self, tokens, targets) -> StepOutput:
        main = torch.cuda.current_stream(self.device)
        start_ev = torch.cuda.Event(enable_timing=self.record_timeline)
        self._tl_start = start_ev if self.record_timeline else None
        if self.iter_done is not None:
            main.wait_event(self.iter_done)
        self.losses.zero_()
        self.step_dev.add_(1)
        start_ev.record(main)
        for st in self.streams.values():
            st.wait_event(start_ev)
        for st in self.opt_streams:
            st.wait_event(start_ev)
        if self.dist is not None:   # before the gradients are zeroed: the peer transport waits there
            self.dist.begin_iteration(self)   # until the partner has read last iteration's gradients
        self._zero_grads()

        done_dirs: dict = {}
        deferred_syncs: list = []
        tl = [] if self.record_timeline else None

        def forward(d, t, x0):
            stream = self.streams[d]
            comp = self.compute[(t.direction, t.stage)]
            mb = t.micro_batch
            if tl is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            res = comp.forward(stream, self.pool, x0=x0, tokens=tokens[mb - 1].reshape(-1),
                               targets=targets[mb - 1].reshape(-1), loss_slot=self.losses[mb - 1:mb])
            if tl is not None:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(stream)
                tl.append((d, t, e0, e1))
            return res

        def backward(d, t, stash, dy):
            stream = self.streams[d]
            if tl is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            wst = self.wstreams.get(d)
            dx, release, release_w = self.compute[(t.direction, t.stage)].backward(
                stream, self.pool, stash, dy, self.ws[d], wstream=wst, dx_dest=self._message_slot(t, live))
            ev = torch.cuda.Event(enable_timing=tl is not None)
            ev.record(stream)
            self.pool.put_all(release, ev, stream)
            done = ev
            if wst is not None:  # join: the task is done when its side-stream wgrads are
                wst.wait_event(ev)
                done = torch.cuda.Event(enable_timing=tl is not None)
                done.record(wst)
                self.pool.put_all(release_w, done, wst)
            if tl is not None:
                tl.append((d, t, e0, done))
            return dx, (ev, done)   # message ready / all of the task's work done

        live: dict = {}
        msgs, stashes = drive(self.order, self.S, self.last_b, forward=forward, backward=backward, stashes=live,
                              send=self._send, recv=self._recv,
                              stage_done=(lambda dr, s, d, ev: self._stage_grads_ready(dr, s, d, ev, done_dirs))
                              if self.eager_sync else (lambda *a: deferred_syncs.append(a)),
                              dev_of=self._dev_of)
        if deferred_syncs:   # w/o eager sync: after all local computation of the device
            dev_end = {}
            for d in self.local_devices:
                wst = self.wstreams.get(d)
                if wst is not None:
                    ev = torch.cuda.Event()
                    ev.record(wst)
                    self.streams[d].wait_event(ev)
                dev_end[d] = torch.cuda.Event()
                dev_end[d].record(self.streams[d])
            for dr, s, d, _ev in sorted(deferred_syncs, key=lambda a: (a[2], self.last_b[a[2]][(a[0], a[1])])):
                self._stage_grads_ready(dr, s, d, dev_end[d], done_dirs)
        if stashes or (msgs and self.dist is None):
            raise RuntimeError(f"protocol violation: {len(stashes)} stashes / {len(msgs)} messages left at flush")
        if self.dist is not None:
            self.dist.end_iteration(self)
        done = torch.cuda.Event()
        done.record(self.opt_stream)
        for st in list(self.streams.values()) + list(self.wstreams.values()) + self.opt_streams[1:]:
            ev = torch.cuda.Event()
            ev.record(st)
            main.wait_event(ev)
        main.wait_event(done)
        if self.dist is not None:
            self.dist.after_join(self, main)
        self.iter_done = torch.cuda.Event()
        self.iter_done.record(main)
        self.timeline = tl
        return StepOutput(self.losses, self.step_count)

    # ---------------------------------------------------------------- messages --
    def _message_slot(self, t, stashes):
        """Co-resident, deferred weight gradients: the input-gradient message
        of backward task ``t`` is the previous stage's output-gradient slot
        of that micro-batch (a weight-gradient GEMM operand), so the producer
        writes it there directly instead of the consumer copying it in."""
        if self.dist is not None or t.stage == 0:
            return None
        prev = self.compute[(t.direction, t.stage - 1)]
        if not prev.defer_wgrad or not prev.plan.halfblocks:
            return None
        pst = stashes.get((t.direction, t.micro_batch, t.stage - 1))
        if pst is None:
            return None
        return prev._buf(pst, ("dy", prev.plan.halfblocks[-1]), self.cfg.hidden, self.pool, None)

    def _send(self, msgs, key, tensor, src, dst, event=None):
        if self.dist is not None and dst != src:
            self.dist.send_msg(self, key, tensor, src, dst)
            return
        if event is None:
            event = torch.cuda.Event()
            event.record(self.streams[src])
        msgs[key] = (tensor, event)

    def _recv(self, msgs, key, d):
        item = msgs.pop(key, None)
        if item is None:
            if self.dist is not None:
                return self.dist.recv_msg(self, key, d)
            raise RuntimeError(f"protocol violation: task on device {d} needs {key} which was never produced")
        tensor, ev = item
        self.streams[d].wait_event(ev)
        return tensor

    # ----------------------------------------------------------- eager sync --
    def _stage_grads_ready(self, dr, s, d, ev, done_dirs):
        if self.dist is not None:
            self.dist.sync_stage(self, dr, s, ev)
            return
        done_dirs.setdefault(s, {})[dr] = ev
        if len(done_dirs[s]) < len(self.dirs):
            return
        st = self.opt_streams[s % len(self.opt_streams)]
        for e in done_dirs[s].values():
            st.wait_event(e)
        grads = [self.stage_params[(x, s)].grad for x in self.dirs]
        outs = list({id(t): t for t in (self.stage_params[(x, s)].flat for x in self.dirs)}.values())  # shared: one
        if s not in self.combined_stages:
            self._adam(s, grads, outs, st)
            return
        # both replicas' GEMM-weight gradients in one set of GEMMs into the
        # first replica's buffer (sum over N micro-batches); AdamW in two
        # parts: the atomically accumulated head averages the two replicas,
        # the GEMM-weight tail reads the combined sum at scale 1/2
        sp0 = self.stage_params[(self.dirs[0], s)]
        self.compute[(self.dirs[0], s)]._deferred_wgrads(st)
        z = sp0.zero_numel
        if z:
            self._adam(s, [g[:z] for g in grads], [o[:z] for o in outs], st, sl=(0, z))
        if z < sp0.numel:
            self._adam(s, [grads[0][z:]], [o[z:] for o in outs], st, grad_scale=0.5, sl=(z, sp0.numel))

    def mean_grads(self) -> dict:
        """{name: fp32 CPU tensor}: the replica-mean gradient AdamW applies
        (tests; synchronises).  Combined deferred weight gradients hold the
        sum over both replicas in the first replica's buffer."""
        if len(self.dirs) == 1:
            return self.gather("grads")
        gd, gu = self.gather("grads", self.dirs[0]), self.gather("grads", self.dirs[1])
        combined = {n for s in self.combined_stages for n in self.stage_params[(self.dirs[0], s)].names}
        return {k: 0.5 * gd[k] if (k in combined and k.endswith(GEMM_WEIGHTS)) else 0.5 * (gd[k] + gu[k])
                for k in gd}

    # ---------------------------------------------------------- introspection --
    def gather(self, what: str = "params", direction: Direction | None = None) -> dict:
        """{name: fp32 CPU tensor} of the local replica's params / grads /
        master weights (tests only; synchronises)."""
        torch.cuda.synchronize(self.device)
        out = {}
        dirs = [direction] if direction is not None else self.dirs
        for (dr, s), sp in self.stage_params.items():
            if dr not in dirs:
                continue
            for n in sp.names:
                if what == "params":
                    t = sp.p[n]
                elif what == "grads":
                    t = sp.g[n]
                elif what == "master":
                    owner = self.opt_owner[s if self.dist is None else (dr, s)]
                    t = owner.master_view(n)
                else:
                    raise ValueError(what)
                out.setdefault(n, t.detach().float().cpu().clone())
        return out

    def measure_task_times(self, reps: int = 7) -> dict:
        """Isolated device time (ms) of every distinct task class of this
        schedule, each timed alone on one stream with CUDA events (median of
        ``reps``) on synthetic inputs:

        * ``(direction, stage, 'F'|'B')``: forward; backward WITH its
          per-micro-batch weight-gradient GEMMs (the paper's B = 2F model);
        * ``(direction, stage, 'Bd')``: backward as the step executes it when
          the stage defers its weight gradients (input-gradient chain only);
        * ``(direction, stage, 'W')``: that replica's deferred weight-gradient
          GEMMs over its n_rep micro-batch slots (K = n_rep M, one GEMM per
          weight), issued at its last backward; 0 for a non-deferring stage."""
        cfg = self.cfg
        M = cfg.micro_batch * cfg.seq
        dev = self.device
        st = torch.cuda.Stream(device=dev)
        tok = torch.randint(0, cfg.vocab, (M,), device=dev, dtype=torch.int32)
        loss = torch.zeros(1, device=dev)
        d0 = self.local_devices[0]
        out = {}
        torch.cuda.synchronize(dev)
        saved = {k: (c.defer_wgrad, c.combined_wgrad, c._fwd_slot, c._bwd_count) for k, c in self.compute.items()}
        # the replay these times feed models one GPU per logical device: time
        # each task with the single-launch GEMM tile model a dedicated GPU
        # uses, not the co-resident throughput pick
        coresident_pick = len(self.local_devices) > 1 and os.environ.get("BP_GEMM_PICK", "") == ""
        if coresident_pick:
            ops.set_option(OPT_GEMM_PICK, 0)

        def fb(comp, s):
            """One forward + backward of ``comp`` on ``st``: (F ms, B ms)."""
            x0 = None if s == 0 else (torch.randn(M, cfg.hidden, device=dev) * 0.1).to(self.dtype)
            dy = None if s == self.S - 1 else (torch.randn(M, cfg.hidden, device=dev) * 1e-3).to(self.dtype)
            torch.cuda.synchronize(dev)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(st)
            stash, msg = comp.forward(st, self.pool, x0=x0, tokens=tok, targets=tok, loss_slot=loss)
            e1.record(st)
            dx, release, _ = comp.backward(st, self.pool, stash, dy, self.ws[d0])
            e2.record(st)
            torch.cuda.synchronize(dev)
            ev = torch.cuda.Event()
            ev.record(st)
            self.pool.put_all([t for t in release if t is not None] + [msg, dx], ev)
            return e0.elapsed_time(e1), e1.elapsed_time(e2)

        def wblock(comp):
            """The replica's deferred weight-gradient GEMMs over its own n_rep slots (ms)."""
            r0 = comp.slot_base * M
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            comp._deferred_wgrads(st, rows=(r0, r0 + comp.n_rep * M))
            e1.record(st)
            torch.cuda.synchronize(dev)
            return e0.elapsed_time(e1)

        # round-robin over the stage replicas, one sample of every task class
        # per round, so clock drift under the power cap spreads over all
        # classes instead of biasing the ones measured during a slow spell;
        # the first round is warm-up, each class reports its median
        samples: dict = {}
        for rnd in range(reps + 1):
            for (dr, s), comp in self.compute.items():
                deferring = saved[(dr, s)][0]
                comp.defer_wgrad = False       # per-micro-batch weight gradients (the paper's task model)
                f, b = fb(comp, s)
                bd, w = b, 0.0
                if deferring:
                    # the executed form: input-gradient chain only (combined_wgrad
                    # keeps backward() from issuing the deferred GEMMs itself) ...
                    comp.defer_wgrad, comp.combined_wgrad = True, True
                    comp._fwd_slot = comp._bwd_count = 0
                    _, bd = fb(comp, s)
                    w = wblock(comp)       # ... and this replica's deferred GEMMs
                    comp.combined_wgrad = saved[(dr, s)][1]
                if rnd:
                    for k, v in (("F", f), ("B", b), ("Bd", bd), ("W", w)):
                        samples.setdefault((dr, s, k), []).append(v)
        for k, v in samples.items():
            v.sort()
            out[k] = v[len(v) // 2]
        for sp in self.stage_params.values():
            sp.grad.zero_()
        for k, c in self.compute.items():
            c.defer_wgrad, c.combined_wgrad, c._fwd_slot, c._bwd_count = saved[k]
        if coresident_pick:
            ops.set_option(OPT_GEMM_PICK, 1)
        return out

    def replay_bubble(self, times: dict, deferred_w: bool = False) -> dict:
        """ASAP replay (reference ``list_schedule``, fusion.py:34-77) of the
        executed per-device orders with the MEASURED task times: the makespan
        and bubble the schedule would have with one GPU per logical device and
        free communication (SPEC.md:263 bubble definition).

        ``deferred_w=False``: the paper's task model, every B carrying its
        micro-batch's weight gradients.  ``deferred_w=True``: the step as it
        executes -- B is the input-gradient chain ('Bd') and each stage
        replica's deferred weight-gradient GEMMs ('W') follow its last
        backward on that device (they fill the pipeline drain); busy time
        includes them."""
        return replay_times(self.sched, times, deferred_w)

    def timeline_spans(self) -> dict:
        """This process's busy time and first-start / last-end (ms, relative
        to the last step's start event) from its per-task CUDA events
        (``record_timeline``); distributed ranks gather these for the
        measured bubble.  Synchronises."""
        torch.cuda.synchronize(self.device)
        if not self.timeline or self._tl_start is None:
            return {"busy_ms": 0.0, "start_ms": 0.0, "end_ms": 0.0, "tasks": 0}
        z = self._tl_start
        iv = sorted((z.elapsed_time(e0), z.elapsed_time(e1)) for _d, _t, e0, e1 in self.timeline)
        busy, cur = 0.0, None   # union of the task intervals (a task's span may overlap the next one's)
        for a, b in iv:
            if cur is None or a > cur[1]:
                if cur is not None:
                    busy += cur[1] - cur[0]
                cur = [a, b]
            else:
                cur[1] = max(cur[1], b)
        busy += cur[1] - cur[0]
        return {"busy_ms": busy, "start_ms": iv[0][0], "end_ms": max(b for _a, b in iv), "tasks": len(iv)}

    def measured_bubble(self):
        """Per-device busy time / makespan from the last step's per-task CUDA
        events and beta = 1 - sum busy / (D * makespan).

        Meaningful in distributed mode (one GPU per logical device); in
        coresident mode the D streams share one GPU and the number only
        describes stream occupancy."""
        if not self.timeline:
            return None
        torch.cuda.synchronize(self.device)
        first = self.timeline[0][2]
        spans: dict = {}
        for d, t, e0, e1 in self.timeline:
            spans.setdefault(d, []).append((first.elapsed_time(e0), first.elapsed_time(e1)))
        busy = {d: sum(b - a for a, b in v) for d, v in spans.items()}
        start = min(a for v in spans.values() for a, _ in v)
        end = max(b for v in spans.values() for _, b in v)
        mk = end - start
        beta = 1 - sum(busy.values()) / (len(spans) * mk) if mk > 0 else 0.0
        return {"busy_ms": busy, "makespan_ms": mk, "bubble": beta}
