"""Peer-memory transport of the multi-GPU train step (no NCCL on the data path).

One process per GPU (or several processes sharing one GPU, the test
configuration), rank == logical device of the schedule.  Everything moves
through the C ABI's peer-memory section (include/bitpipe_comm.h):

Messages (SURVEY §8(e) exchange 1; reference edges schedules.py:181-199)
  Every rank owns a slab of message slots, two per incoming message key
  (kind, direction, micro-batch, destination stage) -- one per iteration
  parity -- and a mailbox of 32-bit flags.  Both are exported once with CUDA
  IPC.  A sender's stream copies the message straight into the receiver's
  slot (copy engine; NVLink via NVSwitch between GPUs) and then sets the
  slot's flag to the iteration number; the receiver's consumer stream waits
  for that value (``cuStreamWaitValue32``).  Slots are tag-addressed, so the
  non-FIFO per-link orders of the reference schedules need
  no receive ordering at all.  Before writing a parity slot again (two
  iterations later) the sender's stream waits for the receiver's
  end-of-iteration flag.

Eager replica-pair sync (SURVEY §8(a) K9
"fused 2-rank peer-read")
  The two holders of model stage s (the down replica on dev_down(s), the up
  replica on D-1-dev_down(s)) export their flat fp32 gradient buffers.
  After its last backward of s, a rank's per-stage optimizer stream raises
  READY[s] in the partner's mailbox, waits for the partner's READY[s], and
  runs ONE fused kernel: AdamW on (g_down + g_up) / 2 where one of the two
  gradients is read from the partner's memory.  Both ranks sum in the same
  fixed order (down first), so their updates are bit-identical
  without any all-reduce.  It then raises READ[s] in the partner's mailbox;
  the partner's next iteration waits for it before overwriting its gradient.

Unlike NCCL, nothing here needs one process per GPU, so the same code runs
with all ranks sharing one B200 (tests/test_gpu_peer.py).
"""
from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from ..schedule import Schedule
from .distributed import DistContext, link_messages
from .lib import check, lib

__all__ = ["PeerContext"]

_HB = 64  # BP_IPC_HANDLE_BYTES


def _export(t: torch.Tensor) -> tuple:
    h = (ctypes.c_ubyte * _HB)()
    off = ctypes.c_size_t()
    check(lib().bp_ipc_export(ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off)), "bp_ipc_export")
    return bytes(h), int(off.value)


def _s(stream) -> ctypes.c_void_p:
    return ctypes.c_void_p(stream.cuda_stream)


class PeerContext(DistContext):
    """Drop-in for :class:`DistContext` (same Trainer hooks) over CUDA IPC
    peer memory and stream-ordered flags."""

    transport = "peer"

    def __init__(self, rank: int, world: int):
        super().__init__(rank, world, cuda=True, replicas=1)
        self._opened: dict = {}     # handle bytes -> imported base address
        self.remote: dict = {}      # rank -> {"mailbox": addr, "slab": addr, "grads": {(dir, s): addr}}
        self.key_index: dict = {}
        self.slot_of: dict = {}
        self.partner: dict = {}     # local stage -> partner rank
        self.senders: list = []
        self.receivers: list = []
        self.flag_sets = self.flag_waits = 0

    # --------------------------------------------------------------- setup --
    def setup(self, trainer) -> None:
        sched: Schedule = trainer.sched
        if sched.D != self.world:
            raise ValueError(f"peer transport needs world == D (world={self.world}, D={sched.D})")
        self.sched = sched
        self.links = link_messages(sched)
        D, S, dev = self.D, sched.num_stages, self.dev
        # mailbox layout: [message flags of every key of the iteration | FREE[D] | READY[S] | READ[S]]
        all_keys = [k for link in sorted(self.links) for k in self.links[link]]
        self.key_index = {k: i for i, k in enumerate(all_keys)}
        self.FREE = len(all_keys)
        self.READY = self.FREE + D
        self.READ = self.READY + S
        cfg = trainer.cfg
        M, h = cfg.micro_batch * cfg.seq, cfg.hidden
        self.msg_shape, self.msg_numel = (M, h), M * h
        self.msg_bytes = M * h * torch.empty(0, dtype=trainer.dtype).element_size()
        incoming = [k for (src, dst) in sorted(self.links) if dst == dev for k in self.links[(src, dst)]]
        self.slot_of = {k: i for i, k in enumerate(incoming)}
        self.senders = sorted({src for (src, dst) in self.links if dst == dev})
        self.receivers = sorted({dst for (src, dst) in self.links if src == dev})
        self.mailbox = torch.zeros(self.READ + S, dtype=torch.int32, device=trainer.device)
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
        torch.cuda.synchronize(trainer.device)
        info = {"rank": self.rank, "mailbox": _export(self.mailbox), "slab": _export(self.slab),
                "slots": {k: i for k, i in self.slot_of.items()},
                "grads": {(dr.value, s): _export(sp.grad) for (dr, s), sp in trainer.stage_params.items()}}
        infos: list = [None] * self.world
        dist.all_gather_object(infos, info)
        need_mb = set(self.senders) | set(self.receivers) | set(self.partner.values())
        for r in sorted(need_mb):
            inf = infos[r]
            rem = {"mailbox": self._open(*inf["mailbox"]), "grads": {}}
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

    # ---------------------------------------------------------- flags --
    def _set(self, stream, addr: int, value: int) -> None:
        check(lib().bp_flag_set(_s(stream), ctypes.c_void_p(addr), value & 0xFFFFFFFF), "bp_flag_set")
        self.flag_sets += 1

    def _wait(self, stream, addr: int, value: int) -> None:
        check(lib().bp_flag_wait(_s(stream), ctypes.c_void_p(addr), value & 0xFFFFFFFF), "bp_flag_wait")
        self.flag_waits += 1

    def _mine(self, i: int) -> int:
        return self.mailbox.data_ptr() + 4 * i

    def _theirs(self, r: int, i: int) -> int:
        return self.remote[r]["mailbox"] + 4 * i

    # ------------------------------------------------- Trainer integration --
    def begin_iteration(self, trainer) -> None:
        self.it = trainer.step_count
        self._free_ok = set()
        if self.it > 1:   # the partner has read last iteration's gradients before they are zeroed
            st = trainer.streams[self.dev]
            for s in sorted(self.partner):
                self._wait(st, self._mine(self.READ + s), self.it - 1)

    def send_msg(self, trainer, key, tensor, src, dst) -> None:
        st = trainer.streams[src]
        par = self.it & 1
        if dst not in self._free_ok:
            if self.it > 2:   # the receiver finished the iteration that last used this parity's slots
                self._wait(st, self._mine(self.FREE + dst), self.it - 2)
            self._free_ok.add(dst)
        rem = self.remote[dst]
        i = rem["slots"][key]
        dst_ptr = rem["slab"] + (2 * i + par) * self.msg_bytes
        if tensor.numel() != self.msg_numel or not tensor.is_contiguous():
            raise RuntimeError(f"peer message {key}: expected a contiguous {self.msg_shape} tensor")
        check(lib().bp_memcpy_async(ctypes.c_void_p(dst_ptr), ctypes.c_void_p(tensor.data_ptr()), self.msg_bytes,
                                    _s(st)), "bp_memcpy_async")
        self._set(st, self._theirs(dst, self.key_index[key]), self.it)
        ev = torch.cuda.Event()
        ev.record(st)
        trainer.pool.put_all([tensor], ev, st)

    def recv_msg(self, trainer, key, d):
        if key not in self.slot_of:
            raise RuntimeError(f"protocol violation: rank {self.rank} has no slot for {key}")
        st = trainer.streams[d]
        self._wait(st, self._mine(self.key_index[key]), self.it)
        return self.slots[(key, self.it & 1)]

    def sync_stage(self, trainer, dr, s, ev) -> None:
        from . import ops
        st = trainer.stage_stream(s)
        st.wait_event(ev)
        sp = trainer.stage_params[(dr, s)]
        owner = trainer.opt_owner[(dr, s)]
        o = trainer.optim
        p = self.partner.get(s)
        if p is None:
            ga, gb = sp.grad.data_ptr(), None
        else:
            self._set(st, self._theirs(p, self.READY + s), self.it)
            self._wait(st, self._mine(self.READY + s), self.it)
            other = [k for k in self.remote[p]["grads"] if k[1] == s]
            if len(other) != 1:
                raise RuntimeError(f"rank {self.rank}: partner {p} exports no gradient of stage {s}")
            peer = self.remote[p]["grads"][other[0]]
            # fixed summation order on both ranks: the first direction's replica first
            down_first = dr == trainer.dirs[0]
            ga, gb = (sp.grad.data_ptr(), peer) if down_first else (peer, sp.grad.data_ptr())
        ops.adam(owner.master, ga, gb, owner.m, owner.v, sp.flat, None, lr=o.lr, beta1=o.beta1, beta2=o.beta2,
                 eps=o.eps, weight_decay=o.weight_decay, step=trainer.step_count, stream=st,
                 step_dev=trainer.step_dev)
        if p is not None:
            self._set(st, self._theirs(p, self.READ + s), self.it)

    def after_join(self, trainer, main) -> None:
        for src in self.senders:
            self._set(main, self._theirs(src, self.FREE + self.dev), self.it)

    def end_iteration(self, trainer) -> None:
        pass
