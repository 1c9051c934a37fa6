"""Multi-GPU plumbing of the train step: one process per GPU, rank == logical
device of the schedule, torch.distributed (NCCL) as the transport.

P2P (activations forward, gradients backward)
  The reference per-device orders are not FIFO-consistent per link (SURVEY
  §0 F5), so messages are tag-addressed: every directed link (src -> dst)
  gets its OWN process group (so the two directions of a device pair never
  serialise on one NCCL stream), the sender issues ``isend`` in its task
  order, and the receiver posts ALL of the iteration's ``irecv``s for that
  link up-front, in the SENDER's order, into slot buffers keyed by
  (kind, direction, micro-batch, destination stage).  A consumer task only
  waits (stream-wise) for its own slot.

Eager gradient synchronisation
  Model stage s lives on dev_down(s) (down replica) and dev_up(s) = D-1-
  dev_down(s) (up replica).  Each (stage) has its own 2-rank group AND its
  own optimizer stream: the two ranks reach their last backwards of their
  shared stages in different orders (BitPipe D=4 N=8 default order: rank 0
  finishes stages [7, 0, 4, 3], rank 3 [4, 3, 7, 0]), and NCCL collectives
  issued on ONE stream would chain (each group's NCCL stream waits for the
  shared stream, which waits for the previous group's collective) into a
  cross-rank cycle.  Right after a rank issues its last backward of s, it
  issues all_reduce(SUM) of that stage's flat fp32 gradient on the stage's
  stream followed by the fused AdamW with grad_scale 1/2 (replica mean).  A
  2-term fp32 sum is commutative, so both replicas compute bit-identical
  updates.  ``sync_order_acyclic`` checks the property that
  makes this deadlock-free for a given schedule.

Data parallelism over W replicated pipelines (``replicated_pipelines``,
core.py:68; "stage replicas co-located"): world = W x D, rank
= w * D + d runs logical device d of pipeline replica w on its own batch;
P2P stays inside a replica, and the stage group spans the stage's holders
in every replica (2W ranks bidirectional, W unidirectional), gradient mean
over all of them.

All of this is host-side control flow; it runs unchanged on CPU tensors with
the gloo backend (``cuda=False``), which is how tests/ exercise it.
"""
from __future__ import annotations

from contextlib import nullcontext

import torch
import torch.distributed as dist

from ..schedule import Schedule, TaskKind

__all__ = ["DistContext", "link_messages", "stage_sync_orders", "sync_order_acyclic"]


def link_messages(sched: Schedule) -> dict:
    """{(src, dst): [key, ...]} -- the cross-device messages of one iteration
    in each sender's production order; key = (kind, direction, mb, dst stage)."""
    last = sched.num_stages - 1
    out: dict = {}
    for src, row in enumerate(sched.per_device):
        for t in row:
            smap = sched.stage_map(t.direction)
            if t.kind is TaskKind.FORWARD and t.stage < last:
                dst = smap.device_of(t.stage + 1)
                key = ("act", t.direction, t.micro_batch, t.stage + 1)
            elif t.kind is TaskKind.BACKWARD and t.stage > 0:
                dst = smap.device_of(t.stage - 1)
                key = ("grad", t.direction, t.micro_batch, t.stage - 1)
            else:
                continue
            if dst != src:
                out.setdefault((src, dst), []).append(key)
    return out


def stage_sync_orders(sched: Schedule) -> dict:
    """{device: [stage, ...]} -- the order in which each logical device
    reaches the eager-sync point (last backward) of its stages."""
    out = {}
    for d, pos in sched.last_backward_positions().items():
        out[d] = [s for (_dr, s), _i in sorted(pos.items(), key=lambda kv: kv[1])]
    return out


def sync_order_acyclic(sched: Schedule, *, shared_stream: bool) -> bool:
    """Can the replica-pair collectives of ``sched`` complete?

    Model: on each device, stage s's collective is issued at its last
    backward.  With ``shared_stream`` (one optimizer stream per rank, NCCL's
    stream semantics) a rank's collectives complete in its issue order, so
    collective s of rank a depends on every collective a issued before it;
    a collective completes only when both members issue it.  The resulting
    wait-for graph over stages must be acyclic.  With one stream per stage
    (what the executor does) there are no such edges and this is trivially
    True."""
    if not shared_stream:
        return True
    orders = stage_sync_orders(sched)
    succ: dict = {}
    for seq in orders.values():
        for a, b in zip(seq, seq[1:]):
            succ.setdefault(a, set()).add(b)
    state: dict = {}

    def cyclic(u) -> bool:
        state[u] = 1
        for w in succ.get(u, ()):
            if state.get(w) == 1 or (state.get(w) is None and cyclic(w)):
                return True
        state[u] = 2
        return False

    return not any(state.get(u) is None and cyclic(u) for u in list(succ))


class DistContext:
    transport = "nccl"

    def __init__(self, rank: int, world: int, *, cuda: bool = True, replicas: int = 1):
        if replicas < 1 or world % replicas:
            raise ValueError(f"world {world} is not a multiple of the pipeline replica count {replicas}")
        self.rank, self.world, self.cuda = rank, world, cuda
        self.replicas = replicas
        self.D = world // replicas
        self.w, self.dev = divmod(rank, self.D)   # pipeline replica, logical device
        self.sched = None
        self.link_group: dict = {}
        self.pair_group: dict = {}
        self.links: dict = {}
        self.slots: dict = {}
        self.inflight: list = []
        self.pending: list = []

    # ----------------------------------------------------------- setup --
    def build_groups(self, sched: Schedule) -> None:
        """Create every group in the same order on every rank."""
        if sched.D != self.D:
            raise ValueError(f"distributed mode needs world == replicas x D "
                             f"(world={self.world}, replicas={self.replicas}, D={sched.D})")
        self.sched = sched
        self.links = link_messages(sched)
        D = self.D
        # every rank creates every group, in one global order (new_group is collective)
        for w in range(self.replicas):
            for (src, dst) in sorted(self.links):
                g = dist.new_group(sorted({w * D + src, w * D + dst}))
                if w == self.w:
                    self.link_group[(src, dst)] = g
        for s in range(sched.num_stages):
            devs = sorted({m.device_of(s) for m in sched.stage_maps})
            members = sorted(w * D + d for w in range(self.replicas) for d in devs)
            if len(members) > 1:
                self.pair_group[s] = (members, dist.new_group(members))
        self.warmup()

    def warmup(self) -> None:
        """Create every communicator up front, in one global order.

        NCCL communicators (and torch's per-pair P2P communicators) are
        created lazily by the first operation, and creation blocks until
        both members arrive.  Posting all receives at iteration start could
        then deadlock (rank a initialising link b->a while rank b
        initialises link a->b).  Walking all groups in the same sorted
        order with a blocking 1-element op makes creation deadlock-free.
        """
        dev = torch.device("cuda", torch.cuda.current_device()) if self.cuda else torch.device("cpu")
        t = torch.zeros(1, device=dev)
        for (src, dst) in sorted(self.link_group):  # links never cross replicas: no inter-replica waits
            g = self.link_group[(src, dst)]
            if self.dev == src:
                dist.send(t, self._g(dst), group=g)
            elif self.dev == dst:
                dist.recv(t, self._g(src), group=g)
        for s in sorted(self.pair_group):
            members, g = self.pair_group[s]
            if self.rank in members:
                dist.all_reduce(t, group=g)
        if self.cuda:
            torch.cuda.synchronize()

    # ------------------------------------------------------- primitives --
    def _g(self, d: int) -> int:
        """Global rank of logical device ``d`` of this rank's pipeline replica."""
        return self.w * self.D + d

    def _sctx(self, stream):
        return torch.cuda.stream(stream) if (self.cuda and stream is not None) else nullcontext()

    def post_recvs(self, alloc, stream=None) -> None:
        """Post every receive of this iteration, per incoming link in the
        sender's order.  ``alloc(key) -> tensor`` provides the slot buffer."""
        with self._sctx(stream):
            for (src, dst), keys in sorted(self.links.items()):
                if dst != self.dev:
                    continue
                g = self.link_group[(src, dst)]
                for key in keys:
                    buf = alloc(key)
                    self.slots[key] = (buf, dist.irecv(buf, self._g(src), group=g))

    def send(self, key, tensor, dst, stream=None) -> None:
        with self._sctx(stream):
            work = dist.isend(tensor, self._g(dst), group=self.link_group[(self.dev, dst)])
        self.inflight.append((tensor, work))

    def recv(self, key, stream=None):
        item = self.slots.pop(key, None)
        if item is None:
            raise RuntimeError(f"protocol violation: rank {self.rank} has no posted receive for {key}")
        buf, work = item
        with self._sctx(stream):
            work.wait()
        return buf

    def allreduce_stage(self, stage: int, tensor, stream=None) -> int:
        """SUM-all-reduce ``tensor`` over every holder of ``stage`` (the other
        direction's replica, and the same stage in the other pipeline
        replicas); returns the number of summed copies (1: nothing to do)."""
        if stage not in self.pair_group:
            return 1
        members, g = self.pair_group[stage]
        with self._sctx(stream):
            if self.cuda:   # NCCL: stream-ordered, the host never blocks
                dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=g)
            else:           # gloo: host-blocking collectives would serialise ranks; run async
                self.pending.append(dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=g, async_op=True))
        return len(members)

    def finish_allreduces(self) -> None:
        for w in self.pending:
            w.wait()
        self.pending.clear()

    def drain_sends(self, stream=None) -> list:
        """Wait (stream-wise) for all sends; returns the sent buffers."""
        out = []
        with self._sctx(stream):
            for t, w in self.inflight:
                w.wait()
                out.append(t)
        self.inflight.clear()
        return out

    # --------------------------------------------- Trainer integration --
    def setup(self, trainer) -> None:
        self.build_groups(trainer.sched)

    def begin_iteration(self, trainer) -> None:
        cfg = trainer.cfg
        shape = (cfg.micro_batch * cfg.seq, cfg.hidden)
        st = trainer.streams[self.dev]
        self.post_recvs(lambda key: trainer.pool.get(shape, trainer.dtype, st), stream=st)

    def send_msg(self, trainer, key, tensor, src, dst) -> None:
        self.send(key, tensor, dst, stream=trainer.streams[src])

    def recv_msg(self, trainer, key, d):
        return self.recv(key, stream=trainer.streams[d])

    def sync_stage(self, trainer, dr, s, ev) -> None:
        st = trainer.stage_stream(s)   # one stream per stage group: no cross-group chaining
        st.wait_event(ev)
        sp = trainer.stage_params[(dr, s)]
        copies = self.allreduce_stage(s, sp.grad, stream=st)
        trainer._adam((dr, s), [sp.grad], [sp.flat], st, grad_scale=1.0 / copies)

    def after_join(self, trainer, main) -> None:
        """Called once every stream of the iteration has joined ``main``."""

    def end_iteration(self, trainer) -> None:
        if self.slots:
            raise RuntimeError(f"protocol violation: {len(self.slots)} posted receives never consumed")
        main = torch.cuda.current_stream(trainer.device)
        sent = self.drain_sends(stream=main)
        ev = torch.cuda.Event()
        ev.record(main)
        trainer.pool.put_all(sent, ev)
