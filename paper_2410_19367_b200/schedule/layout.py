"""Layout engines: ASAP replay of fixed orders, and the greedy fused layout.

``list_schedule`` restates ``pkg/src/pipesched/fusion.py:34-77`` (each device
runs its list in order; a task starts at max(device free, inputs ready)).

``fused_layout`` restates the reference's event-driven bidirectional
co-scheduler (``fusion.py:98-285``) but runs on an *integer tick clock*: with
v chunks per device every forward lasts exactly 1 tick (= 1/v canonical unit)
and every backward 2 ticks, and every clock value the reference can reach
(task ends and defer wake-ups) is a task end, so all times are integers.
Tasks are dense integer ids with per-id attribute arrays instead of objects;
starts are converted back to exact ``Fraction`` canonical units at the end,
which makes the produced orders and slot grids identical to the reference's
(checked byte-for-byte against golden dumps in ``tests/``).

Rules reproduced exactly (they determine the order):
  * dependencies: dataflow, one-at-a-time injection per direction, and the
    unit gate F(mb_j, 0) <- B(first mb of previous unit, gate_stage)
    (``fusion.py:132-153``);
  * priority "unit-1f1b": B -> (-unit, 0, -stage, mb), F -> (-unit, 1, mb,
    stage); "backward-first": (B?0:1, mb, stage) (``fusion.py:186-198``);
  * per clock value, devices are visited 0..D-1 and a started task is
    visible to later devices' defer scans at the same clock;
  * defer: idle until a = end of a running task whenever that task unblocks
    a same-device successor y and max(a+r_y, a+d_y+r_x) < max(now+d_x+r_y,
    now+r_x) (strict), with r = remaining dataflow path (``fusion.py:240-267``);
  * early-forward cap blocks stage-0 injections on the injecting device when
    completed-F minus completed-B chunks would exceed the cap
    (``fusion.py:200-208``).
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass
from fractions import Fraction

from .errors import DeadlockDetected
from .plan import Direction, StageMap, Task, TaskKind

__all__ = ["list_schedule", "FusedLayout", "LayoutPolicy", "fused_layout"]


def list_schedule(per_device, dep_fn, dur_fn) -> dict:
    """ASAP start times for fixed per-device orders.

    ``dep_fn(task)`` yields predecessor tasks (matched by ``.key``) and
    ``dur_fn(task)`` a duration.  Returns ``{task: start}``.  Raises
    :class:`DeadlockDetected` (with the blocked device heads) on a cycle.
    """
    D = len(per_device)
    head = [0] * D
    free = [Fraction(0)] * D
    done_at: dict = {}
    starts: dict = {}
    left = sum(map(len, per_device))
    while left:
        moved = False
        for d in range(D):
            row = per_device[d]
            while head[d] < len(row):
                t = row[head[d]]
                ready = Fraction(0)
                for p in dep_fn(t):
                    end = done_at.get(p.key)
                    if end is None:
                        break
                    if end > ready:
                        ready = end
                else:
                    begin = free[d] if free[d] > ready else ready
                    starts[t] = begin
                    free[d] = done_at[t.key] = begin + dur_fn(t)
                    head[d] += 1
                    left -= 1
                    moved = True
                    continue
                break
        if left and not moved:
            heads = [per_device[d][head[d]] for d in range(D) if head[d] < len(per_device[d])]
            raise DeadlockDetected(f"no runnable task among device heads {heads[:6]!r}",
                                   cycle=heads)
    return starts


@dataclass(frozen=True)
class FusedLayout:
    """Output of :func:`fused_layout`: canonical starts, per-device orders."""

    starts: dict
    per_device: tuple
    makespan: Fraction


@dataclass(frozen=True)
class LayoutPolicy:
    """Greedy-layout knobs (reference ``fusion.py:89-95``).

    ``LayoutPolicy()`` is what the reference builders use.  SURVEY §0 F2:
    ``LayoutPolicy("unit-1f1b", defer=False, gate_stage=g)`` reaches the
    paper's analytic BitPipe bubble for D=2 (any g), D=4 (g=3) and D=8 (g=10).
    """

    priority: str = "unit-1f1b"
    defer: bool = True
    gate_stage: int = 0


_F, _B = 0, 1


def fused_layout(D: int, v: int, maps: dict, micro_batches: dict, *, unit_size: int,
                 early_forward: bool = False, act_cap_chunks: int | None = None,
                 policy: LayoutPolicy = LayoutPolicy()) -> FusedLayout:
    """Greedy co-schedule of one or two pipeline directions on D devices.

    ``maps``: Direction -> StageMap; ``micro_batches``: Direction -> injection
    ordered global ids; ``unit_size``: micro-batches per basic unit per
    direction.  With ``early_forward`` the unit gate is replaced by a
    per-device cap of ``act_cap_chunks`` in-flight chunk activations.
    """
    S = v * D
    # --- dense task table -----------------------------------------------------
    dirs = list(micro_batches)
    kind, mbid, stage, dirn, unit, dev = [], [], [], [], [], []
    base_of: dict = {}            # (dir index, j) -> id of (F, stage 0)
    for di, direction in enumerate(dirs):
        smap = maps[direction].assignment
        for j, mb in enumerate(micro_batches[direction]):
            u = j // unit_size if unit_size else 0
            base_of[(di, j)] = len(kind)
            for s in range(S):
                for k in (_F, _B):
                    kind.append(k)
                    mbid.append(mb)
                    stage.append(s)
                    dirn.append(di)
                    unit.append(u)
                    dev.append(smap[s])
    T = len(kind)

    def tid(di: int, j: int, s: int, k: int) -> int:
        return base_of[(di, j)] + 2 * s + k

    dur = [1 if k == _F else 2 for k in kind]                       # ticks
    rem = [(S - s) + 2 * S if k == _F else 2 * (s + 1)             # ticks
           for k, s in zip(kind, stage)]
    if policy.priority == "unit-1f1b":
        key = [(-u, 0, -s, m) if k == _B else (-u, 1, m, s)
               for k, s, m, u in zip(kind, stage, mbid, unit)]
    else:
        key = [(0 if k == _B else 1, m, s) for k, s, m in zip(kind, stage, mbid)]

    preds: list = [[] for _ in range(T)]
    for di, direction in enumerate(dirs):
        n = len(micro_batches[direction])
        for j in range(n):
            for s in range(S):
                f, b = tid(di, j, s, _F), tid(di, j, s, _B)
                if s > 0:
                    preds[f].append(tid(di, j, s - 1, _F))
                else:
                    if j > 0:
                        preds[f].append(tid(di, j - 1, 0, _F))
                    if not early_forward and unit_size and j >= unit_size:
                        gate_j = (j // unit_size - 1) * unit_size
                        if not 0 <= policy.gate_stage < S:
                            raise KeyError(f"gate_stage {policy.gate_stage} outside 0..{S - 1}")
                        preds[f].append(tid(di, gate_j, policy.gate_stage, _B))
                preds[b].append(tid(di, j, s, _F) if s == S - 1 else tid(di, j, s + 1, _B))
    succs: list = [[] for _ in range(T)]
    for t in range(T):
        for p in preds[t]:
            succs[p].append(t)
    blockers = [len(p) for p in preds]

    inject_dev = [maps[direction].assignment[0] for direction in dirs]
    capped = early_forward and act_cap_chunks is not None
    act = [0] * D

    def cap_blocked(t: int, d: int) -> bool:
        return (capped and kind[t] == _F and stage[t] == 0
                and d == inject_dev[dirn[t]] and act[d] + 1 > act_cap_chunks)

    ready: list = [set() for _ in range(D)]
    for t in range(T):
        if blockers[t] == 0:
            ready[dev[t]].add(t)

    start = [-1] * T
    busy_until = [0] * D
    running: list = []          # heap (end, seq, id)
    clock: list = [0]
    seq = 0
    placed = 0
    while placed < T:
        if not clock:
            stuck = sorted((t for d in range(D) for t in ready[d]), key=key.__getitem__)
            raise DeadlockDetected(f"layout stalled with {T - placed} tasks left",
                                   cycle=[_task_obj(t, kind, mbid, stage, dirn, dirs, unit)
                                          for t in stuck[:6]])
        now = heapq.heappop(clock)
        while clock and clock[0] == now:
            heapq.heappop(clock)
        while running and running[0][0] <= now:
            _, _, t = heapq.heappop(running)
            act[dev[t]] += 1 if kind[t] == _F else -1
            for y in succs[t]:
                blockers[y] -= 1
                if blockers[y] == 0:
                    ready[dev[y]].add(y)

        for d in range(D):
            if busy_until[d] > now or not ready[d]:
                continue
            pick = None
            for t in ready[d]:
                if cap_blocked(t, d):
                    continue
                if pick is None or key[t] < key[pick]:
                    pick = t
            if pick is None:
                continue
            if policy.defer:
                dx, rx = dur[pick], rem[pick]
                horizon = now + dx
                wake = None
                for end_r, _, r in running:
                    if end_r >= horizon:
                        continue
                    for y in succs[r]:
                        if dev[y] != d or blockers[y] != 1 or cap_blocked(y, d):
                            continue
                        a = end_r if end_r > now else now
                        ry, dy = rem[y], dur[y]
                        if max(a + ry, a + dy + rx) < max(now + dx + ry, now + rx):
                            if wake is None or a < wake:
                                wake = a
                if wake is not None and wake > now:
                    heapq.heappush(clock, wake)
                    continue
            ready[d].discard(pick)
            start[pick] = now
            end = now + dur[pick]
            busy_until[d] = end
            seq += 1
            placed += 1
            heapq.heappush(running, (end, seq, pick))
            heapq.heappush(clock, end)

    objs = [_task_obj(t, kind, mbid, stage, dirn, dirs, unit) for t in range(T)]
    starts = {objs[t]: Fraction(start[t], v) for t in range(T)}
    rows = []
    for d in range(D):
        mine = sorted((t for t in range(T) if dev[t] == d), key=start.__getitem__)
        rows.append(tuple(objs[t] for t in mine))
    makespan = Fraction(max((start[t] + dur[t] for t in range(T)), default=0), v)
    return FusedLayout(starts=starts, per_device=tuple(rows), makespan=makespan)


def _task_obj(t, kind, mbid, stage, dirn, dirs, unit) -> Task:
    return Task(TaskKind.FORWARD if kind[t] == _F else TaskKind.BACKWARD,
                mbid[t], stage[t], dirs[dirn[t]], unit[t])
