"""Many iterations of the distributed Trainer over the peer transport with
all ranks sharing cuda:0: exercises every slot parity, the receivers'
end-of-iteration FREE events (iteration >= 3) and the partners' READ events
over a long run; checks finite losses and bit-identical replicas at the end.

  python tools/peer_stress.py [D] [steps] [config]
"""
import io
import os
import socket
import sys
import time

import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, steps, cfg_name, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_19367_b200 import schedule as ps
    from paper_2410_19367_b200.model import CONFIGS, OptimConfig, init_params, synthetic_batch
    from paper_2410_19367_b200.runtime.executor import Trainer
    from paper_2410_19367_b200.runtime.peer import PeerContext
    cfg = CONFIGS[cfg_name]
    sched = ps.build_bitpipe(world, 2 * world, policy=ps.paper_policy(world) if world in ps.PAPER_GATE_STAGE else None)
    ctx = PeerContext(rank, world)
    tr = Trainer(cfg, sched, dtype=torch.bfloat16, optim=OptimConfig(lr=1e-4), params=init_params(cfg, 3),
                 dist_ctx=ctx, device="cuda:0")
    t0 = time.time()
    losses = []
    for step in range(steps):
        tok, tgt = synthetic_batch(cfg, sched.N, seed=100 + step)
        out = tr.train_step(tok.int().cuda(), tgt.int().cuda())
        losses.append(out.losses.float().cpu())
    torch.cuda.synchronize()
    dt = time.time() - t0
    res = {"rank": rank, "losses": torch.stack(losses), "seconds": dt, "host_waits": ctx.host_waits,
           "params": {dr.value: tr.gather("params", dr) for dr in tr.dirs}}
    ctx.close()
    buf = io.BytesIO()
    torch.save(res, buf)
    q.put(buf.getvalue())
    q.close()
    q.join_thread()
    dist.destroy_process_group()


if __name__ == "__main__":
    D = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    cfg = sys.argv[3] if len(sys.argv) > 3 else "small"
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps_ = [ctx.Process(target=worker, args=(r, D, port, steps, cfg, q)) for r in range(D)]
    for p in ps_:
        p.start()
    res = [torch.load(io.BytesIO(q.get(timeout=1800)), weights_only=False) for _ in ps_]
    for p in ps_:
        p.join(timeout=60)
    res.sort(key=lambda r: r["rank"])
    total = sum(r["losses"] for r in res)   # each micro-batch's loss lives on its head rank
    assert torch.isfinite(total).all(), "non-finite loss"
    pd, pu = {}, {}
    for r in res:
        pd.update(r["params"].get("down", {}))
        pu.update(r["params"].get("up", {}))
    same = all(torch.equal(pd[k], pu[k]) for k in pd)
    print(f"D={D} steps={steps} cfg={cfg}: {max(r['seconds'] for r in res):.1f} s, mean loss first "
          f"{total[0].mean():.4f} last {total[-1].mean():.4f}, replicas bit-identical: {same}, host waits "
          f"{[r['host_waits'] for r in res]}")
    assert same
