"""Closed-form bubble ratios and canonical replay metrics.

The reference ships these only as SPEC prose (``SPEC.md:334-342``) and as
the makespan targets of its harness (``pkg/scratch_check.py:41-55``); the
formulas are PAPER Table 2 (``PAPER.md:123-127``) and Appendix B Eq. (2)
(``PAPER.md:487``).  Used by the benchmark to compute the roofline's ideal
bubble and to report the canonical bubble of the order actually executed.
"""
from __future__ import annotations

from fractions import Fraction

from .domain import ApproachId
from .errors import UnsupportedCombination
from .layout import list_schedule
from .plan import Schedule

__all__ = ["analytic_bubble_ratio", "analytic_makespan", "canonical_replay", "canonical_bubble",
           "peak_activations", "search_bitpipe_policy"]


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
