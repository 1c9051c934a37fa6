"""Schedule sweep on GPT-1.3B (BASELINE config 4): BitPipe vs 1F1B vs
interleaved vs Chimera (+ BitPipe-EF, BitPipe F2 paper policy, BitPipe policy search within D M_a)
at D=2/4/8,
N=2D..4D.  For each: 1-GPU co-resident tokens/s, the canonical and analytic
bubble, and the ASAP replay of the executed order with measured task times
(projected makespan / bubble / tokens/s with one GPU per logical device).
Writes one JSON line per config."""
import argparse
import gc
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200 import schedule as ps
from paper_2410_19367_b200.model import CONFIGS, OptimConfig, synthetic_batch
from paper_2410_19367_b200.runtime.executor import Trainer

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="gpt-1.3b")
ap.add_argument("--Ds", default="2,4,8")
ap.add_argument("--mult", default="2,4")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--partition", default="balanced", choices=["balanced", "uniform"])
args = ap.parse_args()
cfg = CONFIGS[args.config]
M = cfg.micro_batch * cfg.seq
for D in map(int, args.Ds.split(",")):
    for k in map(int, args.mult.split(",")):
        N = k * D
        cands = [("bitpipe", lambda: ps.build_bitpipe(D, N)),
                 ("bitpipe-paper-policy", (lambda: ps.build_bitpipe(D, N, policy=ps.paper_policy(D)))
                  if D in ps.PAPER_GATE_STAGE else None),
                 ("bitpipe-policy-search-cap-D", lambda: ps.search_bitpipe_policy(D, N, max_peak=D)[1]),
                 ("bitpipe-early-forward", (lambda: ps.build_bitpipe(D, N, early_forward=True)) if N >= 2 * D else None),
                 ("dapple-1f1b", lambda: ps.build_1f1b(D, N)),
                 ("interleaved-looping", lambda: ps.build_interleaved_looping(D, N, 2)),
                 ("chimera", lambda: ps.build_chimera(D, N))]
        for name, mk in cands:
            if mk is None:
                continue
            sched = mk()
            tr = Trainer(cfg, sched, dtype=torch.bfloat16, optim=OptimConfig(), partition=args.partition)
            tok, tgt = synthetic_batch(cfg, N)
            tok, tgt = tok.int().cuda(), tgt.int().cuda()
            tr.train_step(tok, tgt)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                tr.train_step(tok, tgt)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            rep = tr.replay_bubble(tr.measure_task_times())
            appr = sched.approach
            line = {"approach": name, "D": D, "N": N, "v": sched.v, "partition": tr.partition,
                    "peak_activations_Ma": float(max(ps.peak_activations(sched))),
                    "coresident_1gpu_tokens_per_s": N * M / (ms / 1e3), "ms_per_step_1gpu": ms,
                    "bubble_analytic": float(ps.analytic_bubble_ratio(appr, D, N, sched.v)),
                    "bubble_canonical_order": float(ps.canonical_bubble(sched)),
                    "bubble_replay_measured": rep["bubble"], "replay_makespan_ms": rep["makespan_ms"],
                    "replay_tokens_per_s_D_gpus": N * M / (rep["makespan_ms"] / 1e3)}
            print(json.dumps(line), flush=True)
            del tr
            gc.collect()
            torch.cuda.empty_cache()
