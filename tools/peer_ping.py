"""Token ring over the peer-memory flags: world processes on cuda:0 (or one
per GPU with --per-gpu), rank r waits for flag[it] in its own mailbox, then
copies a small buffer into rank r+1's slot and raises its flag.  Reports the
round-trip time per lap for the stream-memory wait and the polling kernel.

  python tools/peer_ping.py [world] [laps] [stream|spin]
"""
import ctypes
import os
import socket
import sys
import time

import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def log(rank, msg, t0=[time.time()]):
    print(f"[rank {rank} {time.time() - t0[0]:7.2f}s] {msg}", file=sys.stderr, flush=True)


def worker(rank, world, port, laps, mode, q):
    os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    torch.cuda.set_device(0)
    log(rank, "cuda ready")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    log(rank, "gloo ready")
    from paper_2410_19367_b200.runtime.lib import check, lib
    from paper_2410_19367_b200.runtime.peer import _export
    L = lib()
    box = torch.zeros(64, dtype=torch.int32, device="cuda")
    buf = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    infos = [None] * world
    dist.all_gather_object(infos, {"box": _export(box), "buf": _export(buf)})
    nxt = (rank + 1) % world

    def open_(h, off):
        p = ctypes.c_void_p()
        check(L.bp_ipc_open(h, ctypes.byref(p)), "open")
        return p.value + off

    log(rank, "handles exchanged")
    rbox = open_(*infos[nxt]["box"])
    rbuf = open_(*infos[nxt]["buf"])
    st = torch.cuda.Stream()
    s = ctypes.c_void_p(st.cuda_stream)
    wait = L.bp_flag_wait_spin if mode == "spin" else L.bp_flag_wait
    dist.barrier()
    log(rank, "start")
    t0 = time.time()
    for it in range(1, laps + 1):
        if rank != 0 or it > 1:
            check(wait(s, ctypes.c_void_p(box.data_ptr()), it - (rank == 0)), "wait")
        check(L.bp_memcpy_async(ctypes.c_void_p(rbuf), ctypes.c_void_p(buf.data_ptr()), 4096, s), "copy")
        check(L.bp_flag_set(s, ctypes.c_void_p(rbox), it), "set")
    log(rank, "issued")
    ev = torch.cuda.Event()
    ev.record(st)
    t1 = time.time()
    while not ev.query() and time.time() - t1 < 30:
        time.sleep(0.01)
    log(rank, f"done={ev.query()}")
    q.put((rank, ev.query(), time.time() - t0))
    q.close()
    q.join_thread()   # flush before the hard exit
    os._exit(0)


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    laps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    mode = sys.argv[3] if len(sys.argv) > 3 else "stream"
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, world, port, laps, mode, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = []
    for _ in ps:
        try:
            res.append(q.get(timeout=90))
        except Exception:
            break
    for p in ps:
        p.join(timeout=5)
        if p.is_alive():
            p.kill()
    print(f"world {world} laps {laps} mode {mode}: {sorted(res)}")
