"""Multi-process (world_size 2 and 4, gloo, CPU) coverage of the N>1 path.

Each rank runs the product's host-side control flow -- ``executor.drive``
(per-device order, tag-addressed messages, eager-sync launch points) and
``distributed.DistContext`` (per-link groups, receives posted in the
sender's order, per-stage 2-rank all-reduce) -- with the oracle's float64
stage math plugged in as the compute (tests may use the oracle; the product
never does).  The result must equal the sequential baseline: the
schedule-independence theorem of SPEC.md:447 across real processes.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, approach, N, out_q, replicas=1):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import gpt_oracle as O
        from paper_2410_19367_b200 import schedule as ps
        from paper_2410_19367_b200.model import CONFIGS, init_params, synthetic_batch
        from paper_2410_19367_b200.runtime.distributed import DistContext
        from paper_2410_19367_b200.runtime.executor import drive

        cfg = CONFIGS["tiny"]
        oc = O.OracleConfig(cfg.layers, cfg.hidden, cfg.heads, cfg.seq, cfg.vocab, cfg.micro_batch, cfg.causal,
                            lr=1e-3)
        D = world // replicas
        w, dev = divmod(rank, D)
        sched = ps.build(ps.ApproachId(approach), D, N)
        S = sched.num_stages
        hbs = O.stage_halfblocks(cfg.layers, S)
        params = init_params(cfg, 7, perturb=True)
        tok, tgt = synthetic_batch(cfg, N * replicas, seed=11)   # replica w takes micro-batches [w N, (w+1) N)
        tok, tgt = tok[w * N:(w + 1) * N], tgt[w * N:(w + 1) * N]
        dirs = list(sched.directions)
        n_rep = N // len(dirs)
        reps = {d: {k: v.double().clone().requires_grad_(True) for k, v in params.items()} for d in dirs}
        ctx = DistContext(rank, world, cuda=False, replicas=replicas)
        ctx.build_groups(sched)
        ctx.post_recvs(lambda key: torch.empty(cfg.micro_batch, cfg.seq, cfg.hidden, dtype=torch.float64))
        losses = {}

        def forward(d, t, x0):
            P = reps[t.direction]
            if x0 is not None:
                x0 = x0.detach().requires_grad_(True)
            out = O._run_stage(P, hbs[t.stage], x0, oc, first=t.stage == 0, last=t.stage == S - 1,
                               tokens=tok[t.micro_batch - 1], targets=tgt[t.micro_batch - 1])
            if t.stage == S - 1:
                losses[w * N + t.micro_batch] = out.item()
                return (x0, out), None
            return (x0, out), out.detach()

        def backward(d, t, stash, dy):
            x0, out = stash
            if t.stage == S - 1:
                (out / n_rep).backward()
            else:
                out.backward(dy)
            return (x0.grad.detach() if t.stage > 0 else None), None

        def send(msgs, key, tensor, src, dst, event=None):
            if dst == src:
                msgs[key] = tensor
            else:
                ctx.send(key, tensor, dst)

        def recv(msgs, key, d):
            return msgs.pop(key) if key in msgs else ctx.recv(key)

        synced = {}

        def stage_done(dr, s, d, ev):
            names = O_stage_names(cfg, hbs[s], s == 0, s == S - 1)
            P = reps[dr]
            flat = torch.cat([P[n].grad.reshape(-1) for n in names])
            synced[(dr, s)] = (names, flat, ctx.allreduce_stage(s, flat))

        order = [(dev, i, t) for i, t in enumerate(sched.per_device[dev])]
        msgs, stashes = drive(order, S, sched.last_backward_positions(), forward=forward, backward=backward,
                              send=send, recv=recv, stage_done=stage_done,
                              dev_of=lambda dr, s: sched.stage_map(dr).device_of(s))
        ctx.drain_sends()
        ctx.finish_allreduces()
        assert not msgs and not stashes and not ctx.slots
        grads = {}
        for (dr, s), (names, flat, copies) in synced.items():
            flat /= copies
            off = 0
            for n in names:
                k = params[n].numel()
                grads[n] = flat[off:off + k].view_as(params[n]).clone()
                off += k
        out_q.put((rank, losses, {k: v.numpy() for k, v in grads.items()}))
    finally:
        dist.destroy_process_group()


def O_stage_names(cfg, hbs, first, last):
    from paper_2410_19367_b200.model import StagePlan, stage_param_names
    return stage_param_names(StagePlan(0, tuple(hbs), first, last))


@pytest.mark.parametrize("approach,world,N,replicas", [("bitpipe", 2, 4, 1), ("bitpipe", 4, 8, 1),
                                                       ("dapple-1f1b", 2, 4, 1), ("chimera", 4, 4, 1),
                                                       ("bitpipe-early-forward", 2, 4, 1),
                                                       ("bitpipe", 4, 4, 2), ("dapple-1f1b", 4, 4, 2)])
def test_distributed_host_logic_gloo(approach, world, N, replicas):
    """world = replicas x D ranks; with replicas > 1 every pipeline replica
    trains on its own N micro-batches and the stage groups span the replicas
    (data parallelism, core.py:68 replicated_pipelines)."""
    from oracle import gpt_oracle as O
    from paper_2410_19367_b200.model import CONFIGS, init_params, synthetic_batch
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, approach, N, q, replicas)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = CONFIGS["tiny"]
    params = init_params(cfg, 7, perturb=True)
    tok, tgt = synthetic_batch(cfg, N * replicas, seed=11)
    oc = O.OracleConfig(cfg.layers, cfg.hidden, cfg.heads, cfg.seq, cfg.vocab, cfg.micro_batch, cfg.causal)
    seq = O.sequential_baseline(oc, params, tok, tgt)
    losses, grads = {}, {}
    for rank, l, g in results:
        losses.update(l)
        for k, v in g.items():
            v = torch.from_numpy(v)
            if k in grads:   # both replicas of a stage hold the identical synced gradient
                assert torch.equal(grads[k], v)
            grads[k] = v
    assert sorted(losses) == list(range(1, N * replicas + 1))
    for m, v in losses.items():
        assert abs(v - seq.losses[m - 1].item()) < 1e-12
    assert set(grads) == set(params)
    for k in params:
        err = ((grads[k] - seq.grads[k]).norm() / seq.grads[k].norm().clamp_min(1e-300)).item()
        assert err < 1e-9, (k, err)
