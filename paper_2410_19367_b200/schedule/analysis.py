"""Closed-form bubble ratios and canonical replay metrics.

The reference ships these only as SPEC prose (``SPEC.md:334-342``) and as
the makespan targets of its harness (``pkg/scratch_check.py:41-55``); the
formulas are PAPER Table 2 (``PAPER.md:123-127``) and Appendix B Eq. (2)
(``PAPER.md:487``).  Used by the benchmark to compute the roofline's ideal
bubble and to report the canonical bubble of the order actually executed.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction

from .domain import ApproachId, ClusterSpec, ModelProfile, message_size
from .errors import UnsupportedCombination
from .layout import list_schedule
from .plan import Direction, Schedule, TaskKind

__all__ = ["analytic_bubble_ratio", "analytic_makespan", "canonical_replay", "canonical_bubble",
           "peak_activations", "search_bitpipe_policy", "CommTotals", "comm_accounting",
           "analytic_comm_count", "analytic_comm_time", "replay_times", "WeightGradTask"]


def analytic_bubble_ratio(approach: ApproachId, D: int, N: int, v: int = 2) -> Fraction:
    """Table 2 bubble ratio under tb = 2 tf."""
    a = ApproachId(approach)
    if a in (ApproachId.GPIPE, ApproachId.DAPPLE_1F1B):
        return Fraction(D - 1, N + D - 1)
    if a in (ApproachId.INTERLEAVED_LOOPING, ApproachId.V_SHAPED):
        # makespan 3N + 3(D-1)/v over busy 3N
        return 1 - Fraction(3 * N) / (3 * N + Fraction(3 * (D - 1), v))
    if a is ApproachId.CHIMERA:
        return Fraction(D - 2, Fraction(3 * N, 2) + D - 2) if N else Fraction(0)
    if a is ApproachId.BITPIPE:
        return Fraction(D - 2, 3 * N + D - 2)
    if a is ApproachId.BITPIPE_EARLY_FORWARD:
        return Fraction(D - 2, 4 * N + D - 2)
    raise UnsupportedCombination(str(approach))


def analytic_makespan(approach: ApproachId, D: int, N: int, v: int = 2) -> Fraction:
    """Harness targets of ``scratch_check.py:41-55`` in canonical units."""
    a = ApproachId(approach)
    if a in (ApproachId.GPIPE, ApproachId.DAPPLE_1F1B):
        return Fraction(3 * (N + D - 1))
    if a in (ApproachId.INTERLEAVED_LOOPING, ApproachId.V_SHAPED):
        return 3 * N + Fraction(3 * (D - 1), v)
    if a is ApproachId.CHIMERA:
        return Fraction(3 * N + 2 * (D - 2))
    if a is ApproachId.BITPIPE:
        return Fraction(3 * N + (D - 2))
    if a is ApproachId.BITPIPE_EARLY_FORWARD:
        return 3 * N + Fraction(3 * (D - 2), 4)
    raise UnsupportedCombination(str(approach))


def canonical_replay(s: Schedule) -> tuple[dict, Fraction]:
    """ASAP replay of the per-device orders with tf=1, tb=2 (what an ideal
    executor issuing each device's list in order achieves)."""
    starts = list_schedule(s.per_device, s.dependencies, s.canonical_duration)
    makespan = max((st + s.canonical_duration(t) for t, st in starts.items()), default=Fraction(0))
    return starts, makespan


def canonical_bubble(s: Schedule) -> Fraction:
    """1 - sum(busy) / (D * makespan) of the canonical replay."""
    _, mk = canonical_replay(s)
    if mk == 0:
        return Fraction(0)
    busy = sum(s.canonical_duration(t) for t in s.all_tasks())
    return 1 - busy / (s.D * mk)


def peak_activations(s: Schedule) -> list:
    """Per-device peak of in-flight activations in the canonical replay, in
    units of one stage-replica's activations M_a (PAPER Table 2 "peak
    memory"): a chunk forward holds 1/v M_a from its end until
    its backward ends."""
    starts, _ = canonical_replay(s)
    out = []
    for row in s.per_device:
        ev = []
        for t in row:
            end = starts[t] + s.canonical_duration(t)
            ev.append((end, 1 if t.kind.value == "F" else -1))
        live = peak = 0
        for _, dk in sorted(ev, key=lambda e: (e[0], e[1])):  # frees before allocs at equal times
            live += dk
            peak = max(peak, live)
        out.append(Fraction(peak, s.v))
    return out


@dataclass(frozen=True)
class WeightGradTask:
    """Pseudo-task of the as-executed replay: one stage replica's deferred
    weight-gradient GEMMs, after its last backward on its device."""
    stage: int
    direction: Direction

    @property
    def key(self) -> tuple:
        return ("W", self.stage, self.direction)


def replay_times(schedule, times: dict, deferred_w: bool = False) -> dict:
    """ASAP replay of ``schedule``'s per-device orders with measured task
    times ``{(direction, stage, 'F'|'B'|'Bd'|'W'): ms}`` (see
    ``Trainer.measure_task_times`` / ``replay_bubble``).  Integer
    microseconds, exact arithmetic.  Returns makespan, bubble
    beta = 1 - sum busy / (D makespan) and per-device busy."""
    us = {k: Fraction(round(v * 1000)) for k, v in times.items()}   # integer microseconds
    rows = [list(r) for r in schedule.per_device]
    last_b = {}
    if deferred_w:
        for d, pts in schedule.last_backward_positions().items():
            for (dr, st), i in sorted(pts.items(), key=lambda x: -x[1]):
                w = WeightGradTask(st, dr)
                last_b[w.key] = rows[d][i]
                rows[d].insert(i + 1, w)

    def dur(t):
        if isinstance(t, WeightGradTask):
            return us[(t.direction, t.stage, "W")]
        k = t.kind.value
        if deferred_w and k == "B":
            k = "Bd"
        return us[(t.direction, t.stage, k)]

    def deps(t):
        if isinstance(t, WeightGradTask):
            return (last_b[t.key],)
        return schedule.dependencies(t)

    starts = list_schedule(rows, deps, dur)
    mk = max(st + dur(t) for t, st in starts.items())
    busy = [sum(dur(t) for t in row) for row in rows]
    beta = 1 - Fraction(sum(busy)) / (schedule.D * mk)
    return {"makespan_ms": float(mk) / 1000, "bubble": float(beta),
            "busy_ms_per_device": [float(b) / 1000 for b in busy]}


def search_bitpipe_policy(D: int, N: int, v: int = 2, max_peak=None):
    """Generalised F2: over every layout policy of the
    reference engine (``defer`` x ``gate_stage`` over the v*D stages of a
    direction, fusion.py:89-95), the BitPipe order with the lowest canonical
    bubble whose per-device activation peak (``peak_activations``) stays
    within ``max_peak`` M_a (None: no cap); ties go to the lower peak, then
    the lower gate stage.  Returns (policy, schedule, bubble, peak); raises
    ValueError when no policy meets the cap.  Every candidate is a schedule
    of the reference engine (bit-exact under its policy)."""
    from .builders import build_bitpipe
    from .layout import LayoutPolicy

    best = None
    for defer in (False, True):
        for g in range(v * D):
            pol = LayoutPolicy("unit-1f1b", defer=defer, gate_stage=g)
            sch = build_bitpipe(D, N, v, policy=pol)
            peak = max(peak_activations(sch))
            if max_peak is not None and peak > max_peak:
                continue
            key = (canonical_bubble(sch), peak, not defer, g)
            if best is None or key < best[0]:
                best = (key, pol, sch, peak)
    if best is None:
        raise ValueError(f"no BitPipe layout policy keeps the activation peak within {max_peak} M_a")
    return best[1], best[2], best[0][0], best[3]


# -- communication accounting (PAPER Appendix C Table 6)
@dataclass(frozen=True)
class CommTotals:
    """What one iteration of a schedule moves between devices.

    p2p_messages     -- cross-device stage-boundary transfers (activation on
                        F(m,s)->F(m,s+1), gradient on B(m,s+1)->B(m,s));
    local_copies     -- boundaries whose two stages share a device (the V
                        map's fold; "local copying");
    p2p_bytes        -- p2p_messages x message_size (split intra / inter node
                        by the cluster's devices_per_node);
    per_link         -- {(src, dst): messages};
    allreduce_groups -- replica-pair gradient syncs: one per (device pair
                        (d, D-1-d), model stage both hold) for bidirectional
                        schedules -- 2v per pair;
    allreduce_bytes  -- per device: gradient bytes it all-reduces per
                        iteration (grad_bytes_per_stage x stages it holds).
    """
    p2p_messages: int
    local_copies: int
    p2p_bytes: int
    p2p_bytes_intra: int
    p2p_bytes_inter: int
    per_link: dict = field(default_factory=dict)
    allreduce_groups: int = 0
    allreduce_bytes: int = 0


def comm_accounting(s: Schedule, profile: ModelProfile | None = None, cluster: ClusterSpec | None = None,
                    grad_bytes_per_stage: int = 0) -> CommTotals:
    """Count the P2P messages / bytes and allreduce volume of one iteration
    of ``s`` from its dataflow edges (reference ``schedules.py:181-199``) and
    stage maps.  The count for a v=2 interleaved / BitPipe pipeline is the
    looping count minus the local-copy edges: BitPipe moves
    N (4D - 4) messages, interleaved-looping N (4D - 2), 1F1B N (2D - 2)."""
    msg = message_size(profile) if profile is not None else 0
    per_node = cluster.devices_per_node if cluster is not None else max(1, s.D)
    n_msg = n_local = intra = inter = 0
    links: dict = {}
    for t in s.all_tasks():
        if t.kind is TaskKind.FORWARD and t.stage + 1 < s.num_stages:
            nxt = t.stage + 1
        elif t.kind is TaskKind.BACKWARD and t.stage > 0:
            nxt = t.stage - 1
        else:
            continue
        smap = s.stage_map(t.direction)
        src, dst = smap.device_of(t.stage), smap.device_of(nxt)
        if src == dst:
            n_local += 1
            continue
        n_msg += 1
        links[(src, dst)] = links.get((src, dst), 0) + 1
        if src // per_node == dst // per_node:
            intra += msg
        else:
            inter += msg
    groups = 0
    ar_bytes = 0
    if s.is_bidirectional:
        for d in range(s.D):
            held = sum(len(s.stage_map(dr).stages_on(d)) for dr in s.directions)
            groups += held if d < s.D - 1 - d else 0   # every held stage syncs with the partner
            ar_bytes = max(ar_bytes, held * grad_bytes_per_stage)
    return CommTotals(n_msg, n_local, n_msg * msg, intra, inter, links, groups, ar_bytes)


def analytic_comm_count(approach: ApproachId, D: int, N: int) -> int:
    """The message-count factor of PAPER Table 6: the
    number of message times on the critical path of one iteration --
    DAPPLE / Chimera 2N + 2(D-1), 1F1B-Int / BitPipe 4N + 4(D-1)."""
    a = ApproachId(approach)
    if a in (ApproachId.DAPPLE_1F1B, ApproachId.CHIMERA):
        return 2 * N + 2 * (D - 1)
    if a in (ApproachId.INTERLEAVED_LOOPING, ApproachId.BITPIPE):
        return 4 * N + 4 * (D - 1)
    raise UnsupportedCombination(f"Table 6 has no row for {a.value}")


def analytic_comm_time(approach: ApproachId, D: int, N: int, profile: ModelProfile, cluster: ClusterSpec,
                       M_grad: float = 0.0) -> float:
    """PAPER Table 6: count x message_size / W_inter, plus
    M_grad / W_intra for the bidirectional approaches (Chimera, BitPipe)."""
    a = ApproachId(approach)
    t = analytic_comm_count(a, D, N) * message_size(profile) / cluster.inter_node_bandwidth
    if a in (ApproachId.CHIMERA, ApproachId.BITPIPE):
        t += M_grad / cluster.intra_node_bandwidth
    return t
