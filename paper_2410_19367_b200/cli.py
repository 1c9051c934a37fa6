"""``pipesched``-compatible command line.

The reference declares ``pipesched = "pipesched.cli:main"`` but ships no
``cli.py`` (``pkg/pyproject.toml:19-20``); its SPEC fixes the subcommands,
flags and exit codes (``SPEC.md:470-533``).  This is that entry point over
this repo's schedule layer, cost model and (for ``verify --gpu``) the B200
executor:

  plan      write one schedule document (``dump_schedule`` JSON, byte-equal to
            the reference) per approach
  compare   analytic (PAPER Table 2) vs replayed makespan / bubble per approach
  simulate  replay the per-device orders (reference ``list_schedule``) with a
            cost model -> per-task timeline JSON (+ SVG Gantt), report CSV
  search    grid over approach x D x N (x order policy), modelled throughput;
            best row last
  render    ASCII slot grid (``scratch_diag.py``) or SVG Gantt of a schedule
  measure   run the schedule's train step on the B200 (all logical devices
            co-resident) and export the MEASURED per-task timeline (CUDA
            events) in the simulate JSON format, or as an SVG Gantt
  verify    structural checks of every requested schedule (validation,
            acyclicity, byte-determinism, per-link message accounting); with
            ``--gpu`` also schedule independence of the B200 train step in the
            fp32 check mode (every schedule vs the GPipe order, 1e-4)

Exit codes: 0 success, 1 usage / config error, 2 domain error
(builder / simulator), 3 verification failure.  Outputs carry no timestamps
(byte-reproducible).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import sys
from fractions import Fraction

from . import schedule as ps
from .schedule import errors as perr

__all__ = ["main", "build_one", "timeline", "gantt_svg", "ascii_grid"]

EXIT_OK, EXIT_USAGE, EXIT_DOMAIN, EXIT_VERIFY = 0, 1, 2, 3


class UsageError(Exception):
    pass


def build_one(approach: str, D: int, N: int, v: int | None = None, early_forward: bool = False,
              order: str = "default", max_peak=None) -> ps.Schedule:
    """``build`` (builders.py:369-372) with the CLI's naming; ``order='paper'``
    selects the F2 LayoutPolicy order for BitPipe when one is known for D,
    ``order='search'`` the lowest-bubble policy of the reference engine within
    an activation-peak cap (``search_bitpipe_policy``)."""
    try:
        a = ps.ApproachId.parse(approach)
    except Exception as exc:  # unknown approach name -> usage error
        raise UsageError(f"unknown approach {approach!r}") from exc
    if a is ps.ApproachId.BITPIPE and order == "paper":
        if D not in ps.PAPER_GATE_STAGE:
            raise UsageError(f"no paper-policy order known for D={D} (known: {sorted(ps.PAPER_GATE_STAGE)}; "
                             f"use --order search)")
        return ps.build_bitpipe(D, N, v or 2, early_forward, policy=ps.paper_policy(D))
    if a is ps.ApproachId.BITPIPE and order == "search" and not early_forward:
        try:
            return ps.search_bitpipe_policy(D, N, v or 2, max_peak=max_peak)[1]
        except ValueError as exc:
            raise UsageError(str(exc)) from exc
    return ps.build(a, D, N, v, early_forward)


def _durations(sched: ps.Schedule, model: str | None, partition: str):
    """Task duration function: canonical tf = 1, tb = 2 (per chunk 1/v, 2/v;
    schedules.py:165-167), or stage costs of a model config (``model``) under
    the uniform or cost-balanced partition, F = cost, B = 2 x cost."""
    if model is None:
        return sched.canonical_duration, "canonical tf=1, tb=2 (per chunk 1/v, 2/v)"
    from .model import CONFIGS, balanced_counts, stage_costs, stage_partition
    if model not in CONFIGS:
        raise UsageError(f"unknown model {model!r} (known: {sorted(CONFIGS)})")
    cfg = CONFIGS[model]
    counts = (balanced_counts(cfg, sched) if partition == "balanced"
              else [len(p.halfblocks) for p in stage_partition(cfg, sched.num_stages)])
    unit = 1e6
    cost = [Fraction(round(c / unit)) for c in stage_costs(cfg, counts)]
    return (lambda t: cost[t.stage] * (1 if t.kind.value == "F" else 2)), \
        f"{model} stage costs (MFLOP-equivalent per token), {partition} partition {counts}"


def timeline(sched: ps.Schedule, dur) -> dict:
    """ASAP replay of the fixed per-device orders (reference ``list_schedule``,
    fusion.py:34-77): per-task start / end, per-device busy time, makespan and
    bubble 1 - sum busy / (D x makespan)."""
    starts = ps.list_schedule(sched.per_device, sched.dependencies, dur)
    tasks = []
    for d, row in enumerate(sched.per_device):
        for t in row:
            st = starts[t]
            tasks.append({"device": d, "kind": t.kind.value, "micro_batch": t.micro_batch, "stage": t.stage,
                          "direction": t.direction.value, "chunk": t.stage // sched.D,
                          "start": str(st), "end": str(st + dur(t))})
    mk = max((starts[t] + dur(t) for row in sched.per_device for t in row), default=Fraction(0))
    busy = [sum((dur(t) for t in row), Fraction(0)) for row in sched.per_device]
    bubble = 1 - sum(busy) / (sched.D * mk) if mk else Fraction(0)
    return {"approach": sched.approach.value, "D": sched.D, "N": sched.N, "v": sched.v,
            "makespan": str(mk), "bubble": str(bubble), "bubble_float": float(bubble),
            "busy": [str(b) for b in busy], "tasks": tasks}


def ascii_grid(sched: ps.Schedule) -> str:
    """Device x slot grid of the canonical replay (``scratch_diag.py:9-30``):
    one column per 1/v time unit, forward cells ``F<mb><d|u><chunk>``,
    backward cells span two columns, bubbles ``.``."""
    tl = timeline(sched, sched.canonical_duration)
    v = sched.v
    width = int(Fraction(tl["makespan"]) * v)
    rows = [["  .  "] * width for _ in range(sched.D)]
    for t in tl["tasks"]:
        a, b = int(Fraction(t["start"]) * v), int(Fraction(t["end"]) * v)
        tag = f"{t['kind']}{t['micro_batch']}{t['direction'][0]}{t['chunk']}"
        for c in range(a, b):
            rows[t["device"]][c] = f"{tag:<5s}"
    return "\n".join(f"dev{d}: " + "".join(r).rstrip() for d, r in enumerate(rows)) + "\n"


def gantt_svg(tl: dict) -> str:
    """SVG Gantt in the paper's convention: forwards light
    to dark by chunk, backwards a distinct hue, bubbles blank."""
    D = tl["D"]
    mk = float(Fraction(tl["makespan"])) or 1.0
    W, lane, pad = 1200.0, 28, 40
    fwd = ["#cfe3f7", "#8fbce6", "#4f8fd0", "#1f5fa0"]
    bwd = ["#f7d9b8", "#f0b070", "#e08a30", "#b86010"]
    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{int(W + pad + 10)}" height="{D * lane + 40}" '
           f'font-family="monospace" font-size="9">']
    out.append(f'<text x="4" y="14">{tl["approach"]} D={D} N={tl["N"]} v={tl["v"]} '
               f'makespan={tl["makespan"]} bubble={tl["bubble_float"]:.4f}</text>')
    for d in range(D):
        out.append(f'<text x="4" y="{30 + d * lane + 16}">dev{d}</text>')
    for t in tl["tasks"]:
        x0 = pad + W * float(Fraction(t["start"])) / mk
        x1 = pad + W * float(Fraction(t["end"])) / mk
        y = 30 + t["device"] * lane
        pal = fwd if t["kind"] == "F" else bwd
        col = pal[t["chunk"] % len(pal)]
        label = f'{t["micro_batch"]}{t["direction"][0]}'
        out.append(f'<rect x="{x0:.2f}" y="{y}" width="{max(x1 - x0, 0.5):.2f}" height="{lane - 4}" fill="{col}" '
                   f'stroke="#333" stroke-width="0.3"/>')
        if x1 - x0 > 14:
            out.append(f'<text x="{x0 + 2:.2f}" y="{y + 15}">{label}</text>')
    out.append("</svg>")
    return "\n".join(out) + "\n"


def _emit(text: str, out_dir: str | None, name: str):
    if out_dir is None:
        sys.stdout.write(text)
        return
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, name), "w") as f:
        f.write(text)


def _approaches(args) -> list[str]:
    if not args.approach:
        raise UsageError("no --approach given (empty approach list)")
    return args.approach


def _grid_points(args):
    Ds = args.D or [4]
    Ns = args.N or [None]
    for D in Ds:
        for N in Ns:
            yield D, (N if N is not None else 2 * D)


# ------------------------------------------------------------ subcommands --
def cmd_plan(args) -> int:
    for a in _approaches(args):
        for D, N in _grid_points(args):
            s = build_one(a, D, N, args.v, args.early_forward, args.order, args.max_peak)
            name = f"{s.approach.value}_D{D}_N{N}" + ("_paper" if args.order == "paper" else "") + ".json"
            _emit(ps.dump_schedule(s), args.out, name)  # exact dump_schedule bytes
    return EXIT_OK


def _report_rows(args):
    rows = []
    for a in _approaches(args):
        for D, N in _grid_points(args):
            s = build_one(a, D, N, args.v, args.early_forward, args.order, args.max_peak)
            dur, _ = _durations(s, args.model, args.partition)
            tl = timeline(s, dur)
            try:
                ana = ps.analytic_bubble_ratio(s.approach, D, N, s.v)
                ana_s, ana_f = str(ana), f"{float(ana):.6f}"
            except perr.PipeschedError:
                ana_s, ana_f = "", ""
            rows.append({"approach": s.approach.value, "D": D, "N": N, "v": s.v, "order": args.order,
                         "model": args.model or "canonical", "makespan": tl["makespan"],
                         "bubble_sim": tl["bubble"], "bubble_sim_float": f"{tl['bubble_float']:.6f}",
                         "bubble_analytic": ana_s, "bubble_analytic_float": ana_f})
    return rows


def _write_rows(rows, args, name):
    if args.format == "json":
        _emit(json.dumps(rows, indent=1, sort_keys=True) + "\n", args.out, name + ".json")
    else:
        buf = io.StringIO()
        w = csv.DictWriter(buf, fieldnames=list(rows[0].keys()), lineterminator="\n")
        w.writeheader()
        w.writerows(rows)
        _emit(buf.getvalue(), args.out, name + ".csv")


def cmd_compare(args) -> int:
    _write_rows(_report_rows(args), args, "compare")
    return EXIT_OK


def cmd_simulate(args) -> int:
    for a in _approaches(args):
        for D, N in _grid_points(args):
            s = build_one(a, D, N, args.v, args.early_forward, args.order, args.max_peak)
            dur, note = _durations(s, args.model, args.partition)
            tl = timeline(s, dur)
            tl["durations"] = note
            base = f"{s.approach.value}_D{D}_N{N}"
            if args.format == "svg":
                _emit(gantt_svg(tl), args.out, base + ".svg")
            else:
                _emit(json.dumps(tl, indent=1, sort_keys=True) + "\n", args.out, base + ".timeline.json")
    return EXIT_OK


def cmd_search(args) -> int:
    """Grid search (SPEC analysis ``grid_search``, PAPER §4 "grid-searching
    the space of the parameters"): modelled tokens per unit time of every
    (approach, D, N, order) point = N / makespan x D-normalised; the best
    row (lowest makespan per micro-batch per device) is repeated last."""
    rows = []
    orders = ["default", "paper", "search"] if args.order == "both" else [args.order]
    for order in orders:
        args_o = argparse.Namespace(**{**vars(args), "order": order})
        for r in _report_rows(args_o):
            mk = Fraction(r["makespan"])
            r["throughput_per_device"] = f"{float(r['N'] / (mk * r['D'])) if mk else 0.0:.6f}"
            rows.append(r)
    if not rows:
        raise UsageError("empty search space")
    best = max(rows, key=lambda r: float(r["throughput_per_device"]))
    rows.append({**best, "approach": "BEST:" + best["approach"]})
    _write_rows(rows, args, "search")
    return EXIT_OK


def cmd_render(args) -> int:
    for a in _approaches(args):
        for D, N in _grid_points(args):
            s = build_one(a, D, N, args.v, args.early_forward, args.order, args.max_peak)
            if args.format == "svg":
                _emit(gantt_svg(timeline(s, s.canonical_duration)), args.out, f"{s.approach.value}_D{D}_N{N}.svg")
            else:
                _emit(ascii_grid(s), args.out, f"{s.approach.value}_D{D}_N{N}.txt")
    return EXIT_OK


def _verify_structure(s: ps.Schedule) -> list[str]:
    fails = []
    try:
        ps.validate_schedule(s)
    except perr.PipeschedError as exc:
        fails.append(f"validate_schedule: {exc}")
    text = ps.dump_schedule(s)
    if ps.dump_schedule(ps.load_schedule(text)) != text:
        fails.append("dump/load round trip is not byte-identical")
    # every cross-device boundary message is produced once and consumed once
    sent, recv = {}, {}
    for d, row in enumerate(s.per_device):
        for t in row:
            m = s.stage_map(t.direction)
            last = m.num_stages - 1
            if t.kind.value == "F" and t.stage < last and m.device_of(t.stage + 1) != d:
                sent[("act", t.direction, t.micro_batch, t.stage + 1)] = d
            if t.kind.value == "B" and t.stage > 0 and m.device_of(t.stage - 1) != d:
                sent[("grad", t.direction, t.micro_batch, t.stage - 1)] = d
            if t.kind.value == "F" and t.stage > 0 and m.device_of(t.stage - 1) != d:
                recv[("act", t.direction, t.micro_batch, t.stage)] = d
            if t.kind.value == "B" and t.stage < last and m.device_of(t.stage + 1) != d:
                recv[("grad", t.direction, t.micro_batch, t.stage)] = d
    if set(sent) != set(recv):
        fails.append(f"unmatched P2P messages: {len(set(sent) ^ set(recv))}")
    try:
        timeline(s, s.canonical_duration)
    except perr.PipeschedError as exc:
        fails.append(f"replay: {exc}")
    return fails


def cmd_verify(args) -> int:
    failed = 0
    lines = []
    scheds = []
    for a in _approaches(args):
        for D, N in _grid_points(args):
            s = build_one(a, D, N, args.v, args.early_forward, args.order, args.max_peak)
            scheds.append(s)
            fails = _verify_structure(s)
            # byte-determinism: an independent rebuild dumps the same bytes
            rebuilt = build_one(a, D, N, args.v, args.early_forward, args.order, args.max_peak)
            if ps.dump_schedule(rebuilt) != ps.dump_schedule(s):
                fails.append("rebuild is not byte-identical")
            failed += bool(fails)
            lines.append(f"{'FAIL' if fails else 'ok  '} structure {s.approach.value} D={D} N={N}"
                         + ("" if not fails else ": " + "; ".join(fails)))
    if args.gpu:
        failed += _verify_gpu(scheds, lines, args)
    sys.stdout.write("\n".join(lines) + "\n")
    return EXIT_VERIFY if failed else EXIT_OK


def _verify_gpu(scheds, lines, args) -> int:
    """Schedule independence of the B200 train step: in the
    fp32 check mode every schedule's per-micro-batch losses and replica-mean
    gradients equal those of the GPipe order on the same batch (1e-4)."""
    import torch

    from .model import CONFIGS, OptimConfig, init_params, synthetic_batch
    from .runtime.executor import Trainer
    cfg = CONFIGS[args.model or "tiny"]
    failed = 0
    refs = {}
    for s in scheds:
        params = init_params(cfg, args.seed, perturb=True)
        tok, tgt = synthetic_batch(cfg, s.N, seed=args.seed + 1)
        if s.N not in refs:
            ref_tr = Trainer(cfg, ps.build(ps.ApproachId.GPIPE, 2, s.N), dtype=torch.float32,
                             optim=OptimConfig(lr=1e-3), params=params)
            out = ref_tr.train_step(tok.int().cuda(), tgt.int().cuda())
            refs[s.N] = (out.losses.double().cpu(), ref_tr.gather("grads"))
        tr = Trainer(cfg, s, dtype=torch.float32, optim=OptimConfig(lr=1e-3), params=params)
        out = tr.train_step(tok.int().cuda(), tgt.int().cuda())
        if s.is_bidirectional:
            grads = tr.mean_grads()
        else:
            grads = tr.gather("grads")
        rl, rg = refs[s.N]

        def rel(a, b):
            a, b = a.double().cpu(), b.double().cpu()
            return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()

        le = rel(out.losses, rl)
        ge = max(rel(grads[k], rg[k]) for k in rg)
        bad = not (le < 1e-4 and ge < 1e-4)
        failed += bad
        lines.append(f"{'FAIL' if bad else 'ok  '} gpu {s.approach.value} D={s.D} N={s.N}: loss err {le:.2e}, "
                     f"grad err {ge:.2e} vs gpipe D=2")
    return failed


def cmd_measure(args) -> int:
    """Measured timeline of one train step (after warm-up) of ``--model`` on
    this GPU: per-task start / end in ms from the CUDA events the executor
    records on each logical device's stream, per-device busy time, makespan
    and bubble (with co-resident logical devices the bubble
    describes stream occupancy, not idle GPU time)."""
    import torch
    if not torch.cuda.is_available():
        raise perr.PipeschedError("measure needs a CUDA device")
    from .model import CONFIGS, OptimConfig, synthetic_batch
    from .runtime.executor import Trainer
    model = args.model or "tiny"
    if model not in CONFIGS:
        raise UsageError(f"unknown model {model!r} (known: {sorted(CONFIGS)})")
    cfg = CONFIGS[model]
    for a in _approaches(args):
        for D, N in _grid_points(args):
            s = build_one(a, D, N, args.v, args.early_forward, args.order, args.max_peak)
            tr = Trainer(cfg, s, dtype=torch.bfloat16 if args.dtype == "bf16" else torch.float32,
                         optim=OptimConfig(), record_timeline=True, partition=args.partition)
            tok, tgt = synthetic_batch(cfg, N, seed=args.seed)
            tok, tgt = tok.int().cuda(), tgt.int().cuda()
            for _ in range(3):
                tr.train_step(tok, tgt)
            torch.cuda.synchronize()
            first = tr.timeline[0][2]
            tasks, busy = [], [0.0] * D
            for d, t, e0, e1 in tr.timeline:
                a0, a1 = first.elapsed_time(e0), first.elapsed_time(e1)
                busy[d] += a1 - a0
                tasks.append({"device": d, "kind": t.kind.value, "micro_batch": t.micro_batch, "stage": t.stage,
                              "direction": t.direction.value, "chunk": t.stage // D,
                              "start": f"{a0:.4f}", "end": f"{a1:.4f}"})
            t0 = min(float(x["start"]) for x in tasks)
            mk = max(float(x["end"]) for x in tasks) - t0
            for x in tasks:
                x["start"], x["end"] = f"{float(x['start']) - t0:.4f}", f"{float(x['end']) - t0:.4f}"
            bubble = 1 - sum(busy) / (D * mk) if mk else 0.0
            tl = {"approach": s.approach.value, "D": D, "N": N, "v": s.v, "unit": "ms", "model": model,
                  "partition": tr.partition, "makespan": f"{mk:.4f}", "bubble": f"{bubble:.6f}",
                  "bubble_float": bubble, "busy": [f"{b:.4f}" for b in busy], "tasks": tasks,
                  "durations": "measured (CUDA events per task on each logical device's stream; co-resident)"}
            base = f"{s.approach.value}_D{D}_N{N}_measured"
            if args.format == "svg":
                _emit(gantt_svg(tl), args.out, base + ".svg")
            else:
                _emit(json.dumps(tl, indent=1, sort_keys=True) + "\n", args.out, base + ".timeline.json")
    return EXIT_OK


def make_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="pipesched", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name, fn, fmt in (("plan", cmd_plan, ["json"]), ("compare", cmd_compare, ["csv", "json"]),
                          ("simulate", cmd_simulate, ["json", "svg"]), ("search", cmd_search, ["csv", "json"]),
                          ("render", cmd_render, ["txt", "svg"]), ("verify", cmd_verify, ["txt"]),
                          ("measure", cmd_measure, ["json", "svg"])):
        p = sub.add_parser(name)
        p.set_defaults(fn=fn)
        p.add_argument("--approach", action="append", help="approach name or alias (repeatable)")
        p.add_argument("--D", type=int, action="append", help="devices (repeatable)")
        p.add_argument("--N", type=int, action="append", help="micro-batches (repeatable; default 2D)")
        p.add_argument("--v", type=int, default=None)
        p.add_argument("--early-forward", choices=["on", "off"], default="off")
        p.add_argument("--order", choices=["default", "paper", "search"] + (["both"] if name == "search" else []),
                       default="default", help="BitPipe order policy (paper = SURVEY §0 F2 gate table; search = "
                                               "lowest-bubble reference-engine policy within --max-peak)")
        p.add_argument("--max-peak", type=float, default=None,
                       help="activation cap for --order search, in M_a per device (PAPER Table 2: D)")
        p.add_argument("--model", default=None, help="cost model config (gpt-1.3b, bert-large, ...); "
                                                     "default canonical tf=1, tb=2")
        p.add_argument("--partition", choices=["uniform", "balanced"], default="uniform")
        p.add_argument("--out", default=None, help="output directory (default stdout)")
        p.add_argument("--format", choices=fmt, default=fmt[0])
        p.add_argument("--seed", type=int, default=7)
        if name == "verify":
            p.add_argument("--gpu", action="store_true", help="also run the B200 train-step equivalence suite")
        if name == "measure":
            p.add_argument("--dtype", choices=["bf16", "fp32"], default="bf16")
    return ap


def main(argv=None) -> int:
    ap = make_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as exc:  # argparse usage errors exit 2; the SPEC wants 1
        return EXIT_OK if exc.code == 0 else EXIT_USAGE
    args.early_forward = args.early_forward == "on"
    try:
        return args.fn(args)
    except UsageError as exc:
        sys.stderr.write(f"pipesched: usage error: {exc}\n")
        return EXIT_USAGE
    except perr.PipeschedError as exc:
        sys.stderr.write(f"pipesched: {type(exc).__name__}: {exc}\n")
        return EXIT_DOMAIN


if __name__ == "__main__":
    sys.exit(main())
