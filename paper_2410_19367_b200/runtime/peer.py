"""Peer-memory transport of the multi-GPU train step (no NCCL on the data path).

One process per GPU (or several processes sharing one GPU, the test
configuration), rank == logical device of the schedule, all ranks on one
node.  Data moves through CUDA IPC peer memory (include/bitpipe_comm.h
``bp_ipc_*`` / ``bp_memcpy_async``); every cross-rank ORDER is a CUDA IPC
event, so CUDA sees each dependency -- the north star's "CUDA-event-gated
P2P activation and gradient send/recv".

Messages (SURVEY §8(e) exchange 1; reference edges schedules.py:181-199)
  Every rank owns a slab of message slots, two per incoming message key
  (kind, direction, micro-batch, destination stage) -- one per iteration
  parity -- exported once.  A sender's stream copies the message straight
  into the receiver's slot (copy engine; NVLink via NVSwitch between GPUs)
  and records the key's interprocess event; the receiver's stream waits on
  that event.  Slots are tag-addressed, so the non-FIFO per-link orders of
  the reference schedules need no receive ordering.  Before a
  parity slot is written again (two iterations later) the sender's stream
  waits on the receiver's end-of-iteration event.

Eager replica-pair sync (SURVEY §8(a) K9
"fused 2-rank peer-read")
  The two holders of model stage s export their flat fp32 gradients.  After
  its last backward of s, a rank's per-stage stream records READY[s]; once
  the partner's READY[s] is recorded it waits on it and runs ONE fused
  kernel: AdamW on (g_down + g_up) / 2 with one of the two gradients read
  from the partner's memory.  Both ranks sum in the same fixed order (down
  first), so their updates are bit-identical without any
  all-reduce.  It then records READ[s]; the partner's next iteration waits on
  it before overwriting its gradient.

Why events and a host handshake, not stream-memory flags
  A stream waiting on another process's event only waits for the event's
  LAST RECORD at the time of the wait call, so the waiting host must know
  the record has been issued.  Each producer therefore bumps a counter in
  a node-local shared-memory block right after issuing the record (hosts
  run ahead of the GPUs, so these host waits are short).  A previous
  version gated streams with cuStreamWaitValue32 flags: those dependencies
  are invisible to CUDA, and a per-stage stream blocked on its partner's
  flag stalled the rank's compute stream (measured: a D=4 step that never
  finished, while the same step without that wait ran in 0.1 s) -- the
  deadlock the CUDA driver documentation warns about for ordering not
  expressed through CUDA-visible dependencies.  The flags remain in the C
  ABI for pure-C hosts that can guarantee it.

Host-side ordering is deadlock-free: a host blocks only on (i) a message
its device's list needs (the schedule's own acyclic dataflow), (ii) the
previous iteration's READ / FREE handshakes, and (iii) at the end of its
task list, partners' READY records still missing -- while its list is in
progress a missing READY only defers the issue of that stage's update.
"""
from __future__ import annotations

import ctypes
import time

import torch
import torch.distributed as dist

from ..schedule import Schedule
from .distributed import DistContext, link_messages
from .lib import check, lib

__all__ = ["PeerContext"]

_HB = 64  # BP_IPC_HANDLE_BYTES
_TIMEOUT_S = 600.0


def _export(t: torch.Tensor) -> tuple:
    h = (ctypes.c_ubyte * _HB)()
    off = ctypes.c_size_t()
    check(lib().bp_ipc_export(ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off)), "bp_ipc_export")
    return bytes(h), int(off.value)


def _ipc_event() -> torch.cuda.Event:
    return torch.cuda.Event(interprocess=True)


class PeerContext(DistContext):
    """Drop-in for :class:`DistContext` (same Trainer hooks) over CUDA IPC
    peer memory, interprocess events and a shared-memory host handshake."""

    transport = "peer"

    def __init__(self, rank: int, world: int):
        super().__init__(rank, world, cuda=True, replicas=1)
        self._opened: dict = {}     # handle bytes -> imported base address
        self.remote: dict = {}      # rank -> {"slab": addr, "slots": {...}, "grads": {(dir, s): addr}}
        self.key_index: dict = {}
        self.slot_of: dict = {}
        self.partner: dict = {}     # local stage -> partner rank
        self.senders: list = []
        self.receivers: list = []
        self.pending: list = []     # stage syncs waiting for the partner's READY record
        self.host_waits = 0
        self._shm = None

    # --------------------------------------------------------------- setup --
    def setup(self, trainer) -> None:
        import socket
        from multiprocessing import resource_tracker, shared_memory

        import numpy as np
        sched: Schedule = trainer.sched
        if sched.D != self.world:
            raise ValueError(f"peer transport needs world == D (world={self.world}, D={sched.D})")
        self.sched = sched
        self.links = link_messages(sched)
        D, S, dev = self.D, sched.num_stages, self.dev
        all_keys = [k for link in sorted(self.links) for k in self.links[link]]
        self.key_index = {k: i for i, k in enumerate(all_keys)}
        cfg = trainer.cfg
        M, h = cfg.micro_batch * cfg.seq, cfg.hidden
        self.msg_shape, self.msg_numel = (M, h), M * h
        self.msg_bytes = M * h * torch.empty(0, dtype=trainer.dtype).element_size()
        incoming = [k for (src, dst) in sorted(self.links) if dst == dev for k in self.links[(src, dst)]]
        outgoing = [k for (src, dst) in sorted(self.links) if src == dev for k in self.links[(src, dst)]]
        self.slot_of = {k: i for i, k in enumerate(incoming)}
        self.senders = sorted({src for (src, dst) in self.links if dst == dev})
        self.receivers = sorted({dst for (src, dst) in self.links if src == dev})
        self.slab = torch.empty(max(1, 2 * len(incoming)) * M * h, dtype=trainer.dtype, device=trainer.device)
        self.slots = {}
        for k, i in self.slot_of.items():
            for par in (0, 1):
                v = self.slab[(2 * i + par) * M * h:(2 * i + par + 1) * M * h].view(M, h)
                self.slots[(k, par)] = v
                trainer.pool.foreign.add(v.data_ptr())
        for s in range(S):
            holders = sorted({m.device_of(s) for m in sched.stage_maps})
            if dev in holders and len(holders) == 2:
                self.partner[s] = holders[0] if holders[1] == dev else holders[1]
        # interprocess events, two parities each: per outgoing message, per
        # local paired stage READY / READ, and this rank's end-of-iteration FREE
        self.ev_msg = {self.key_index[k]: (_ipc_event(), _ipc_event()) for k in outgoing}
        self.ev_ready = {s: (_ipc_event(), _ipc_event()) for s in self.partner}
        self.ev_read = {s: (_ipc_event(), _ipc_event()) for s in self.partner}
        self.ev_free = (_ipc_event(), _ipc_event())
        # host handshake counters: [message keys | READY[rank][S] | READ[rank][S] | FREE[rank]]
        self.C_READY = len(all_keys)
        self.C_READ = self.C_READY + self.world * S
        self.C_FREE = self.C_READ + self.world * S
        n_counters = self.C_FREE + self.world
        name = None
        if self.rank == 0:
            self._shm = shared_memory.SharedMemory(create=True, size=8 * n_counters)
            name = self._shm.name
        torch.cuda.synchronize(trainer.device)
        hs = lambda pair: [e.ipc_handle() for e in pair]  # noqa: E731
        info = {"rank": self.rank, "host": socket.gethostname(), "shm": name, "device": trainer.device.index,
                "slab": _export(self.slab), "slots": dict(self.slot_of),
                "grads": {(dr.value, s): _export(sp.grad) for (dr, s), sp in trainer.stage_params.items()},
                "ev_msg": {i: hs(p) for i, p in self.ev_msg.items()},
                "ev_ready": {s: hs(p) for s, p in self.ev_ready.items()},
                "ev_read": {s: hs(p) for s, p in self.ev_read.items()},
                "ev_free": hs(self.ev_free)}
        infos: list = [None] * self.world
        dist.all_gather_object(infos, info)
        if len({i["host"] for i in infos}) != 1:
            raise RuntimeError("peer transport: all ranks must run on one node (CUDA IPC, shared memory)")
        if self.rank != 0:
            # attach WITHOUT registering with the resource tracker (Python 3.12
            # registers attaches too, and would unlink rank 0's segment when
            # this process exits); rank 0 owns and unlinks it
            reg = resource_tracker.register
            resource_tracker.register = lambda *a, **k: None
            try:
                self._shm = shared_memory.SharedMemory(name=infos[0]["shm"])
            finally:
                resource_tracker.register = reg
        self.cnt = np.ndarray((n_counters,), dtype=np.int64, buffer=self._shm.buf)
        if self.rank == 0:
            self.cnt[:] = 0
        # an interprocess event is opened on its EXPORTER's device (as torch's
        # own CUDA IPC does); a stream may wait on an event of another device
        def opn(r, hl):
            dev = torch.device("cuda", infos[r]["device"])
            return tuple(torch.cuda.Event.from_ipc_handle(dev, x) for x in hl)

        self.in_msg = {}
        for k in incoming:
            i = self.key_index[k]
            src = next(r for r in self.senders if i in infos[r]["ev_msg"])
            self.in_msg[i] = opn(src, infos[src]["ev_msg"][i])
        self.p_ready = {s: opn(p, infos[p]["ev_ready"][s]) for s, p in self.partner.items()}
        self.p_read = {s: opn(p, infos[p]["ev_read"][s]) for s, p in self.partner.items()}
        self.r_free = {r: opn(r, infos[r]["ev_free"]) for r in self.receivers}
        torch.cuda.set_device(trainer.device)   # (opening may have switched the current device)
        for r in sorted(set(self.receivers) | set(self.partner.values())):
            inf = infos[r]
            rem = {"grads": {}}
            if r in self.receivers:
                rem["slab"] = self._open(*inf["slab"])
                rem["slots"] = inf["slots"]
            if r in self.partner.values():
                rem["grads"] = {k: self._open(*v) for k, v in inf["grads"].items()}
            self.remote[r] = rem
        torch.cuda.synchronize(trainer.device)
        dist.barrier()

    def _open(self, handle: bytes, offset: int) -> int:
        base = self._opened.get(handle)
        if base is None:
            p = ctypes.c_void_p()
            check(lib().bp_ipc_open(handle, ctypes.byref(p)), "bp_ipc_open")
            base = self._opened[handle] = int(p.value)
        return base + offset

    def close(self) -> None:
        """Unmap every imported buffer (after the device is idle), then wait
        for all ranks so no exporter frees memory a peer still maps."""
        torch.cuda.synchronize()
        for base in self._opened.values():
            check(lib().bp_ipc_close(ctypes.c_void_p(base)), "bp_ipc_close")
        self._opened.clear()
        self.remote.clear()
        dist.barrier()
        if self._shm is not None:
            self.cnt = None
            self._shm.close()
            if self.rank == 0:
                self._shm.unlink()
            self._shm = None

    # ------------------------------------------------------ host handshake --
    def _publish(self, idx: int, value: int) -> None:
        self.cnt[idx] = value

    def _await(self, idx: int, value: int) -> None:
        """Block the host until counter ``idx`` reaches ``value`` (its
        producer has issued the matching event record)."""
        if self.cnt[idx] >= value:
            return
        self.host_waits += 1
        t0 = time.monotonic()
        while self.cnt[idx] < value:
            if time.monotonic() - t0 > _TIMEOUT_S:
                raise RuntimeError(f"peer transport: rank {self.rank} waited {_TIMEOUT_S:.0f} s for counter {idx} "
                                   f">= {value} (a peer rank died or the schedules differ)")
            time.sleep(0)

    # ------------------------------------------------- Trainer integration --
    def begin_iteration(self, trainer) -> None:
        self.it = trainer.step_count
        self.par = self.it & 1
        self._free_ok = set()
        if self.it > 1:   # the partner has read last iteration's gradients before they are zeroed
            st = trainer.streams[self.dev]
            S = self.sched.num_stages
            for s, p in sorted(self.partner.items()):
                self._await(self.C_READ + p * S + s, self.it - 1)
                st.wait_event(self.p_read[s][(self.it - 1) & 1])

    def send_msg(self, trainer, key, tensor, src, dst) -> None:
        self._try_pending(trainer)
        st = trainer.streams[src]
        if dst not in self._free_ok:
            if self.it > 2:   # the receiver finished the iteration that last used this parity's slots
                self._await(self.C_FREE + dst, self.it - 2)
                st.wait_event(self.r_free[dst][self.par])
            self._free_ok.add(dst)
        rem = self.remote[dst]
        i = rem["slots"][key]
        dst_ptr = rem["slab"] + (2 * i + self.par) * self.msg_bytes
        if tensor.numel() != self.msg_numel or not tensor.is_contiguous():
            raise RuntimeError(f"peer message {key}: expected a contiguous {self.msg_shape} tensor")
        check(lib().bp_memcpy_async(ctypes.c_void_p(dst_ptr), ctypes.c_void_p(tensor.data_ptr()), self.msg_bytes,
                                    ctypes.c_void_p(st.cuda_stream)), "bp_memcpy_async")
        k = self.key_index[key]
        self.ev_msg[k][self.par].record(st)
        self._publish(k, self.it)
        ev = torch.cuda.Event()
        ev.record(st)
        trainer.pool.put_all([tensor], ev, st)

    def recv_msg(self, trainer, key, d):
        if key not in self.slot_of:
            raise RuntimeError(f"protocol violation: rank {self.rank} has no slot for {key}")
        self._try_pending(trainer)
        k = self.key_index[key]
        self._await(k, self.it)
        trainer.streams[d].wait_event(self.in_msg[k][self.par])
        return self.slots[(key, self.par)]

    def sync_stage(self, trainer, dr, s, ev) -> None:
        st = trainer.stage_stream(s)
        st.wait_event(ev)
        p = self.partner.get(s)
        if p is None:
            self._update(trainer, dr, s, st)
            return
        self.ev_ready[s][self.par].record(st)
        self._publish(self.C_READY + self.rank * self.sched.num_stages + s, self.it)
        self.pending.append((dr, s))
        self._try_pending(trainer)

    def _try_pending(self, trainer, block: bool = False) -> None:
        S = self.sched.num_stages if self.sched is not None else 0
        keep = []
        for dr, s in self.pending:
            idx = self.C_READY + self.partner[s] * S + s
            if block:
                self._await(idx, self.it)
            elif self.cnt[idx] < self.it:
                keep.append((dr, s))
                continue
            st = trainer.stage_stream(s)
            st.wait_event(self.p_ready[s][self.par])
            self._update(trainer, dr, s, st)
            self.ev_read[s][self.par].record(st)
            self._publish(self.C_READ + self.rank * S + s, self.it)
        self.pending = keep

    def _update(self, trainer, dr, s, st) -> None:
        """Fused replica-mean AdamW of stage s (peer-read of the partner's
        gradient in a fixed down-first order), or plain AdamW unpaired."""
        from . import ops
        sp = trainer.stage_params[(dr, s)]
        owner = trainer.opt_owner[(dr, s)]
        o = trainer.optim
        p = self.partner.get(s)
        if p is None:
            ga, gb = sp.grad.data_ptr(), None
        else:
            other = [k for k in self.remote[p]["grads"] if k[1] == s]
            if len(other) != 1:
                raise RuntimeError(f"rank {self.rank}: partner {p} exports no gradient of stage {s}")
            peer = self.remote[p]["grads"][other[0]]
            down_first = dr == trainer.dirs[0]
            ga, gb = (sp.grad.data_ptr(), peer) if down_first else (peer, sp.grad.data_ptr())
        ops.adam(owner.master, ga, gb, owner.m, owner.v, sp.flat, None, lr=o.lr, beta1=o.beta1, beta2=o.beta2,
                 eps=o.eps, weight_decay=o.weight_decay, step=trainer.step_count, stream=st,
                 step_dev=trainer.step_dev)

    def end_iteration(self, trainer) -> None:
        self._try_pending(trainer, block=True)

    def after_join(self, trainer, main) -> None:
        self.ev_free[self.par].record(main)
        self._publish(self.C_FREE + self.rank, self.it)
