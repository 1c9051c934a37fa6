#!/usr/bin/env python
"""BitPipe train-step benchmark (one JSON line on rank 0).

Workload (BASELINE.json metric "GPT tokens/sec/box ... (frac of roofline);
bubble fraction"): GPT-1.3B (24 layers, h=2048, s=2048, V=50304, B=1),
BitPipe v=2, N=16 micro-batches per iteration (global batch 16 x 2048
tokens), bf16 compute with fp32 master weights / AdamW.

  --gpus 1 : the flagship D=8 schedule with all 8 logical devices
             co-resident on GPU 0 (one CUDA stream each).
  --gpus n : one process per GPU (torchrun), D = n logical devices, same
             N = 16 micro-batches -> fixed total work ("strong" scaling).

``value`` is tokens/s with inputs already in HBM; ``e2e`` is the same step
through the public ``Trainer.train_step`` API with the tokens copied from
pinned host memory and the per-micro-batch losses read back every step.
``--impl reference`` times the CPU restatement of the train step (the
reference has no numeric implementation) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GPT tokens/sec/box at D=1/2/4/8 B200 (frac of roofline); bubble fraction"
# ncu --set full, fc1 forward GEMM 2048x8192x2048 as the co-resident step issues it
# (bias + GELU + saved pre-activation, 256-wide pair tiles, L2 hints; tools/gemm_ncu_fc1.py,
# profiles/r2b_ncu_fc1_summary.txt, mean of 3 launches): dram__bytes_read.sum +
# dram__bytes_write.sum per launch
TRAFFIC_FC1_BYTES = 42.154e6 + 20.088e6


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="gpt-1.3b")
    ap.add_argument("--layers", type=int, default=None,
                    help="reduced-depth slice of --config at full width (e.g. --config gpt-10b --layers 8)")
    ap.add_argument("--approach", default="bitpipe")
    ap.add_argument("--D", type=int, default=None)
    ap.add_argument("--N", type=int, default=16)
    ap.add_argument("--order", default="paper", choices=["paper", "default", "search"],
                    help="BitPipe order: 'paper' = the F2 LayoutPolicy order (SURVEY §0 F2; bit-exact vs the "
                         "reference engine under that policy; reaches the analytic bubble) where one is known for "
                         "D, else the policy search; 'search' = lowest-bubble reference-engine policy within "
                         "--max-peak; 'default' = build_bitpipe's default policy")
    ap.add_argument("--max-peak", type=float, default=None, help="activation cap (M_a per device) for --order search")
    ap.add_argument("--paper-policy", action="store_true", help="alias of --order paper")
    ap.add_argument("--replicas", type=int, default=1,
                    help="data-parallel pipeline replicas W (N>1 only): D = world / W, each replica on its own batch")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dump-task-times", default=None,
                    help="write the measured per-(direction, stage, kind) task times (ms) and the partition as JSON")
    ap.add_argument("--partition", default="auto", choices=["auto", "calibrated", "balanced", "uniform"],
                    help="layer -> stage split (model.resolve_partition): 'calibrated' = measured B200 cost table "
                         "of the config, replayed as executed (model.calibrated_counts); 'balanced' = FLOP cost "
                         "model (model.balanced_counts); 'auto' = calibrated when the config has a table")
    return ap.parse_args()


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            with open(self.path) as f:
                for line in f:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def plan(args, D):
    """(approach, layout policy, schedule) of the benchmarked configuration."""
    from paper_2410_19367_b200 import schedule as ps
    N = args.N
    approach = ps.ApproachId.parse(args.approach)
    policy = None
    if approach is ps.ApproachId.BITPIPE and args.order != "default":
        if (args.order == "paper" or args.paper_policy) and D in ps.PAPER_GATE_STAGE and args.max_peak is None:
            policy = ps.paper_policy(D)
        else:
            policy = ps.search_bitpipe_policy(D, N, 2, max_peak=args.max_peak)[0]
    if approach in (ps.ApproachId.BITPIPE, ps.ApproachId.BITPIPE_EARLY_FORWARD):
        sched = ps.build_bitpipe(D, N, 2, approach is ps.ApproachId.BITPIPE_EARLY_FORWARD, policy=policy)
    else:
        sched = ps.build(approach, D, N)
    return approach, policy, sched


def workload_config(cfg, args, approach, policy, sched, G, W):
    """The ``config`` object of the JSON line (identical for both arms)."""
    from paper_2410_19367_b200.model import load_calibration, resolve_partition
    D, N = sched.D, sched.N
    counts = resolve_partition(cfg, sched, args.partition)
    M = cfg.micro_batch * cfg.seq
    weights_gb = 2 * cfg.n_params() / 1e9
    act_gb = N * M * cfg.hidden * 2 * 14 * cfg.layers / 1e9 / max(1, G)
    return {"workload": f"{cfg.name} {approach.value} v=2 D={D} N={N}"
                        + (f" (layout policy gate {policy.gate_stage})" if policy else "")
                        + (" all logical devices co-resident on 1 GPU" if G == 1 else " one rank per GPU"),
            "global_batch": W * N * cfg.micro_batch, "seq_len": cfg.seq, "layers": cfg.layers,
            "hidden": cfg.hidden, "vocab": cfg.vocab,
            "parallelism": f"pp{D} bidirectional" + (f" x dp{W}" if W > 1 else ""),
            "partition": {"kind": ("calibrated" if load_calibration(cfg.name) is not None else "balanced")
                          if args.partition == "auto" else args.partition, "halfblocks_per_stage": counts},
            "l2": f"inputs larger than L2: {weights_gb:.1f} GB bf16 weights + ~{act_gb:.1f} GB of stashed "
                  f"activations per GPU per step vs 126 MB L2 (no flush needed)"}


def reference_arm(args):
    """The reference's CPU path for the benchmarked configuration: the
    oracle's CPU restatement of the train step (the reference has no numeric
    implementation) on a bounded sample per step, plus the
    schedule build (the reference's own CPU code, timed through the bit-exact
    port) -- rank 0 only."""
    import torch
    from oracle.gpt_oracle import OracleConfig, layer_sample_seconds
    from paper_2410_19367_b200.model import CONFIGS, flops_per_token

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = _model_config(args)
    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    D = args.D or (args.gpus // args.replicas if args.gpus > 1 else 8)
    approach, policy, sched = plan(args, D)
    t0 = time.perf_counter()
    plan(args, D)
    build_ms = (time.perf_counter() - t0) * 1e3
    oc = OracleConfig(cfg.layers, cfg.hidden, cfg.heads, cfg.seq, cfg.vocab, cfg.micro_batch, cfg.causal)
    M = cfg.micro_batch * cfg.seq
    layer_flops = 3.0 * (24 * cfg.hidden ** 2 + 4 * cfg.seq * cfg.hidden) * M
    scale = flops_per_token(cfg) * M / layer_flops  # sample -> one micro-batch through the whole model
    for _ in range(max(1, args.warmup)):
        layer_sample_seconds(oc)
    times = [layer_sample_seconds(oc) for _ in range(max(1, args.steps))]
    t = statistics.median(times)
    value = M / (t * scale)
    W = args.replicas
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": len(times), "warmup": max(1, args.warmup), "ms_per_step": t * scale * args.N * W * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(cfg, args, approach, policy, sched, args.gpus, W),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port",
                         "sample": f"each step: fwd+bwd of 1 transformer layer on 1 micro-batch ({M} tokens), fp32 "
                                   f"torch CPU (oracle restatement of SPEC run_schedule_numeric), extrapolated by "
                                   f"model FLOPs (x{scale:.1f}) to whole-model tokens/s; ms_per_step = the "
                                   f"extrapolated full step",
                         "schedule_build_ms": build_ms},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _self_launch(args) -> int:
    """``--gpus N`` without a torchrun environment: launch N ranks (one
    process per GPU) through torch.distributed.run on this node and return
    its exit code; rank 0 prints the JSON line."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def _model_config(args):
    """BASELINE config by name, optionally at reduced depth (same width)."""
    import dataclasses
    from paper_2410_19367_b200.model import CONFIGS
    cfg = CONFIGS[args.config]
    if args.layers is not None and args.layers != cfg.layers:
        cfg = dataclasses.replace(cfg, name=f"{cfg.name}-L{args.layers}", layers=args.layers)
    return cfg


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_self_launch(args))
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import torch.distributed as dist
    from paper_2410_19367_b200 import schedule as ps
    from paper_2410_19367_b200.model import CONFIGS, OptimConfig, flops_per_token, synthetic_batch
    from paper_2410_19367_b200.runtime import ops
    from paper_2410_19367_b200.runtime.executor import Trainer, replay_times

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    # BP_SHARE_GPU=1: every rank on cuda:0 -- a functional test of the
    # multi-rank path (transport, max-over-ranks timing, measured bubble) on a
    # one-GPU box; its timings are NOT multi-GPU numbers (time-sliced GPU)
    shared = os.environ.get("BP_SHARE_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    cfg = _model_config(args)
    dist_ctx = None
    transport = os.environ.get("BP_TRANSPORT", "peer" if args.replicas == 1 else "nccl")
    if world > 1:
        if transport == "peer":   # CUDA IPC peer memory + interprocess events; gloo for the handle exchange
            from paper_2410_19367_b200.runtime.peer import PeerContext
            dist.init_process_group("gloo")
            dist_ctx = PeerContext(rank, world)
        else:                     # NCCL P2P + per-stage 2-rank all-reduce
            from paper_2410_19367_b200.runtime.distributed import DistContext
            dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device(f"cuda:{local}"))
            dist_ctx = DistContext(rank, world, replicas=args.replicas)
        D = dist_ctx.D
    else:
        D = args.D or 8
    N = args.N
    approach, policy, sched = plan(args, D)
    tr = Trainer(cfg, sched, dtype=torch.bfloat16, optim=OptimConfig(), dist_ctx=dist_ctx, partition=args.partition)
    W = dist_ctx.replicas if dist_ctx is not None else 1
    tok, tgt = synthetic_batch(cfg, N, seed=1234 + (dist_ctx.w if dist_ctx is not None else 0))  # replica's batch
    tok_h = tok.int().pin_memory()
    tgt_h = tgt.int().pin_memory()
    tok_d, tgt_d = tok_h.cuda(), tgt_h.cuda()
    main_stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        tr.train_step(tok_d, tgt_d)
    barrier()
    # co-resident (1 process): the step is captured once as a CUDA graph and
    # replayed (BP_GRAPH=0: eager launches).  Measured: BERT-large D=4 N=8
    # +1.5-2.5 % (the host enqueues ~13 us per launch, ~43 ms per 58 ms
    # step), GPT-1.3B +0.4 %
    graphed = world == 1 and os.environ.get("BP_GRAPH", "1") == "1"
    if graphed:  # capture one iteration as a CUDA graph (one more warm-up step), replay it in the timed region
        l0 = ops.launch_count()
        tr.train_step(tok_d, tgt_d)
        torch.cuda.synchronize()
        tr.enable_graph()
        tr.train_step(tok_d, tgt_d)   # capture + first replay
        torch.cuda.synchronize()
        launches_per_step = (ops.launch_count() - l0) // 2
    launches0 = ops.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(main_stream)
        for _ in range(args.steps):
            out = tr.train_step(tok_d, tgt_d)
        ev1.record(main_stream)
        barrier()
    launches = ops.launch_count() - launches0
    if graphed:  # replays launch on the device without passing through the host wrappers
        launches = launches_per_step * args.steps
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:   # device time, max over ranks
        t = torch.tensor([ms])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    tokens_per_step = W * N * cfg.micro_batch * cfg.seq   # whole job: every pipeline replica
    value = tokens_per_step / (ms / 1e3)
    loss_mean = out.losses.float().mean().item()

    # ---- end to end through the public API: H2D inputs + D2H losses per step
    e2e = None
    if not args.no_e2e:
        barrier()
        t0 = time.perf_counter()
        e2e_steps = max(3, args.steps // 2)
        for _ in range(e2e_steps):
            td = tok_h.to("cuda", non_blocking=True)
            gd = tgt_h.to("cuda", non_blocking=True)
            o = tr.train_step(td, gd)
            host_losses = o.losses.to("cpu")
        barrier()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
        if world > 1:
            t = torch.tensor([e2e_ms])
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = t.item()
        e2e = {"value": tokens_per_step / (e2e_ms / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": tok_h.numel() * 4 + tgt_h.numel() * 4,
               "d2h_bytes_per_step": host_losses.numel() * 4, "ms_per_step": e2e_ms}

    # ---- bubble of the executed order under the measured task times
    replay = None
    measured = None
    if world == 1:
        times = tr.measure_task_times()
        if args.dump_task_times:
            with open(args.dump_task_times, "w") as f:
                json.dump({"config": cfg.name, "D": D, "N": N, "partition": [len(p.halfblocks) for p in tr.plans],
                           "times": [[str(k[0].value), k[1], k[2], v] for k, v in sorted(
                               times.items(), key=lambda x: (x[0][0].value, x[0][1], x[0][2]))]}, f, indent=0)
        replay = tr.replay_bubble(times)
        replay["tokens_per_s_on_D_gpus"] = tokens_per_step / (replay["makespan_ms"] / 1e3)
        replay["task_model"] = "paper: every B carries its micro-batch's weight gradients"
        if tr.deferred_stages:
            rx = tr.replay_bubble(times, deferred_w=True)
            rx["tokens_per_s_on_D_gpus"] = tokens_per_step / (rx["makespan_ms"] / 1e3)
            rx["task_model"] = ("as executed: B = input-gradient chain, each stage replica's deferred "
                                "weight-gradient GEMMs (K = n_rep M) after its last backward")
            unit = {k: (1.0 if k[2] == "F" else 2.0 if k[2] == "B" else 1.0 if k[2] == "Bd" else N / len(sched.directions))
                    for k in times}
            rx["canonical"] = replay_times(sched, unit, deferred_w=True)["bubble"]
            replay["as_executed"] = rx
    else:
        # one more step with per-task CUDA events on every rank (relative to a
        # start event recorded right after a barrier), gathered to rank 0:
        # beta = 1 - sum_d busy_d / (D * makespan)
        barrier()
        tr.record_timeline = True
        tr.train_step(tok_d, tgt_d)
        torch.cuda.synchronize()
        tr.record_timeline = False
        spans = tr.timeline_spans()
        allspans = [None] * world
        dist.all_gather_object(allspans, spans)
        busy = sum(x["busy_ms"] for x in allspans)
        t0 = min(x["start_ms"] for x in allspans)
        t1 = max(x["end_ms"] for x in allspans)
        measured = {"bubble": 1 - busy / (world * (t1 - t0)), "makespan_ms": t1 - t0,
                    "busy_ms_per_rank": [x["busy_ms"] for x in allspans],
                    "how": "per-task CUDA events on each rank's compute + weight-gradient streams, one extra step, "
                           "times relative to a per-rank start event recorded after a barrier"}

    # ---- roofline: whole step and the dominant kernel (tcgen05 GEMM)
    peak_burst, peak_sust, hbm, peak_kind = _peaks()
    F_tok = flops_per_token(cfg)
    G = max(world, 1)
    beta_ideal = float(ps.analytic_bubble_ratio(approach, D, N)) if G > 1 else 0.0
    roof_tps = G * peak_sust * 1e12 * (1 - beta_ideal) / F_tok
    beta_order = float(ps.canonical_bubble(sched))
    beta_default_order = (float(ps.canonical_bubble(ps.build_bitpipe(D, N))) if approach is ps.ApproachId.BITPIPE
                          else beta_order)
    # dominant kernel: the tcgen05 GEMM.  Live: CUDA events around every GEMM
    # launch (on its own stream) during one extra step after the timed region,
    # with the logical devices' work serialised on one stream so that a
    # launch's span is its own device time (in the concurrent step the spans
    # overlap other streams' kernels).  Serialised step time is reported too.
    Mtok = cfg.micro_batch * cfg.seq
    # (distributed: each rank's compute and weight-gradient streams serialised
    # likewise; its per-stage optimizer streams only run AdamW)
    tr.disable_graph()  # the probe times each launch through the host wrappers
    tr.streams = {d: main_stream for d in tr.streams}
    tr.wstreams = {}  # weight-gradient GEMMs serialised too (their spans would include cross-stream waits)
    if world == 1:
        tr.opt_stream, tr.opt_streams = main_stream, [main_stream]  # and the combined ones + AdamW
    tr.train_step(tok_d, tgt_d)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ops.gemm_probe_start()
    s0.record(main_stream)
    tr.train_step(tok_d, tgt_d)
    s1.record(main_stream)
    torch.cuda.synchronize()
    probes = ops.gemm_probe_stop()
    serial_ms = s0.elapsed_time(s1)
    gemm_flops = sum(p[0] for p in probes)
    gemm_ms = sum(p[2].elapsed_time(p[3]) for p in probes)
    n_gemm = len(probes)
    achieved = gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else 0.0
    gemm_share = gemm_ms / serial_ms if serial_ms > 0 else 0.0
    fc1 = [p for p in probes if p[1] == (Mtok, cfg.ffn, cfg.hidden)]
    fc1_us = 1e3 * sum(p[2].elapsed_time(p[3]) for p in fc1) / max(1, len(fc1))

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": G, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform token ids, seed 1234; random-init "
                                                            "weights N(0,0.02))",
            "config": workload_config(cfg, args, approach, policy, sched, G, W),
            "loss_mean": loss_mean,
            "e2e": e2e,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_sust, "unit": "TFLOP/s",
                         "frac": achieved / peak_sust,
                         "traffic": TRAFFIC_FC1_BYTES,
                         "kernel": "bp::gemm_tc2_kernel (tcgen05 2-SM GEMM), all launches of one step "
                                   "(logical devices serialised on one stream, events per launch)",
                         "serial_step_ms": serial_ms,
                         "launches": n_gemm, "avg_launch_us": 1e3 * gemm_ms / max(1, n_gemm),
                         "algorithmic_flops_per_launch": gemm_flops / max(1, n_gemm),
                         "share_of_step": gemm_share, "fc1_fprop_avg_us": fc1_us,
                         "peak_kind": f"{peak_kind} sustained (kernel timed inside a long step)",
                         "traffic_note": "dram read+write bytes per fc1-fprop launch from ncu --set full "
                                         "(profiles/r2b_ncu_fc1_summary.txt): 42.2 MB read + 20.1 MB written; "
                                         "the launch's algorithmic bytes are 109 MB (X 8 MiB + W 32 MiB read, "
                                         "GELU output + pre-activation 2 x 32 MiB written): the pre-activation "
                                         "streams to DRAM (L2 evict_first), the GELU output is still in the "
                                         "126 MB L2 when the launch ends -- no wasted re-reads"},
            "step_roofline": {"tokens_per_s": roof_tps, "frac": value / roof_tps, "F_tok": F_tok,
                              "peak_tflops": peak_sust, "peak_kind": f"{peak_kind} sustained",
                              "beta_ideal": beta_ideal, "model_tflops": value * F_tok / 1e12},
            "bubble": {"analytic": float(ps.analytic_bubble_ratio(approach, D, N)),
                       "canonical_of_order": beta_order,
                       "order": (f"layout policy defer={policy.defer} gate_stage={policy.gate_stage}"
                                 + (" (F2 paper gate)" if ps.PAPER_GATE_STAGE.get(D) == policy.gate_stage
                                    and not policy.defer else "")) if policy else "reference default",
                       "peak_activations_Ma": float(max(ps.peak_activations(sched))),
                       "canonical_of_reference_default_order": beta_default_order,
                       "measured_replay": replay,
                       "measured": measured,
                       "note": "1 GPU: the D logical devices share the GPU, so pipeline bubbles are filled by other "
                               "streams; measured_replay = ASAP replay of the executed per-device orders with each "
                               "task's isolated measured device time (one GPU per logical device, free comm); "
                               "as_executed: the same with the deferred weight gradients as separate drain tasks "
                               "(canonical = F 1, B 1, W 1 per micro-batch)"},
            "gpu_launches": launches,
            "wgrad": {"deferred_stages": tr.deferred_stages, "combined_stages": sorted(tr.combined_stages),
                      "note": "deferred = one K = N M weight-gradient GEMM per weight at the stage's last "
                              "backward; the rest per micro-batch (slots over the memory budget)"},
            "transport": (dist_ctx.transport if dist_ctx is not None else "co-resident (stream events)")
                         + (" -- ALL RANKS SHARE ONE GPU (BP_SHARE_GPU=1): functional test, not a multi-GPU number"
                            if shared else ""),
            "launch": "CUDA graph replay of the captured step" if graphed else "eager launches",
            "clocks": clocks,
        }
        if rank == 0 and os.environ.get("BP_SKIP_CPU_BASELINE") != "1":
            line["cpu_baseline"] = _cpu_baseline(cfg, args)
        print(json.dumps(line), flush=True)
    if world > 1:
        if hasattr(dist_ctx, "close"):
            dist_ctx.close()
        dist.destroy_process_group()


def _cpu_baseline(cfg, args):
    import torch
    from oracle.gpt_oracle import OracleConfig, layer_sample_seconds
    from paper_2410_19367_b200.model import flops_per_token
    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    oc = OracleConfig(cfg.layers, cfg.hidden, cfg.heads, cfg.seq, cfg.vocab, cfg.micro_batch, cfg.causal)
    M = cfg.micro_batch * cfg.seq
    layer_flops = 3.0 * (24 * cfg.hidden ** 2 + 4 * cfg.seq * cfg.hidden) * M
    scale = flops_per_token(cfg) * M / layer_flops
    layer_sample_seconds(oc)
    t = statistics.median(layer_sample_seconds(oc) for _ in range(3))
    return {"value": M / (t * scale), "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"fwd+bwd of 1 transformer layer, 1 micro-batch ({M} tokens), fp32 torch CPU (oracle "
                      f"restatement of SPEC run_schedule_numeric), extrapolated x{scale:.1f} by model FLOPs"}


if __name__ == "__main__":
    main()
