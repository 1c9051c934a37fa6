"""Does a stream blocked in a flag wait stall OTHER streams of its process?
Two processes on cuda:0.  Rank 1: stream A waits on a flag that rank 0 only
raises after a 3 s host sleep; meanwhile stream B (independent) runs small
kernels and writes progress markers into pinned host memory.  Rank 1
reports B's progress 1.5 s in (should be complete) and after the flag.

  python tools/peer_block.py [stream|spin]
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


def worker(rank, port, mode, q):
    os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from paper_2410_19367_b200.runtime.lib import check, lib
    from paper_2410_19367_b200.runtime.peer import _export
    L = lib()
    box = torch.zeros(64, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    infos = [None] * 2
    dist.all_gather_object(infos, _export(box))
    p = ctypes.c_void_p()
    check(L.bp_ipc_open(infos[1 - rank][0], ctypes.byref(p)), "open")
    rbox = p.value + infos[1 - rank][1]
    nst = int(os.environ.get("N_STREAMS", "2"))
    pool = [torch.cuda.Stream() for _ in range(nst)]
    b, a = pool[0], pool[int(os.environ.get("A_INDEX", "1"))]
    prog = torch.zeros(4, dtype=torch.int32, pin_memory=True)
    x = torch.randn(1024, 1024, device="cuda")
    with torch.cuda.stream(b):
        x = x * 1.0001   # warm the kernel before timing
    check(L.bp_flag_set(ctypes.c_void_p(b.cuda_stream), ctypes.c_void_p(prog.data_ptr() + 8), 1), "warm")
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.time()
    out = {}
    if rank == 0:
        time.sleep(5.0)
        check(L.bp_flag_set(ctypes.c_void_p(a.cuda_stream), ctypes.c_void_p(rbox), 1), "set")
        torch.cuda.synchronize()
    else:
        wait = L.bp_flag_wait_spin if mode == "spin" else L.bp_flag_wait
        if os.environ.get("BLOCK_EVENT") == "1":   # A first waits for an event of B (the stage-sync pattern)
            with torch.cuda.stream(b):
                x = x * 1.0001
            ev0 = torch.cuda.Event()
            ev0.record(b)
            a.wait_event(ev0)
        check(wait(ctypes.c_void_p(a.cuda_stream), ctypes.c_void_p(box.data_ptr()), 1), "wait")
        check(L.bp_flag_set(ctypes.c_void_p(a.cuda_stream), ctypes.c_void_p(prog.data_ptr()), 7), "markA")
        with torch.cuda.stream(b):
            for i in range(1, 101):
                x = x * 1.0001
                check(L.bp_flag_set(ctypes.c_void_p(b.cuda_stream), ctypes.c_void_p(prog.data_ptr() + 4), i), "mB")
        time.sleep(1.5)
        out["t"] = time.time() - t0
        out["B_at_1.5s"] = int(prog[1])
        out["A_at_1.5s"] = int(prog[0])
        torch.cuda.synchronize()
        out["B_end"] = int(prog[1])
        out["A_end"] = int(prog[0])
    q.put((rank, out))
    q.close()
    q.join_thread()
    os._exit(0)


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "stream"
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, port, mode, q)) for r in range(2)]
    for p_ in ps:
        p_.start()
    res = [q.get(timeout=60) for _ in ps]
    for p_ in ps:
        p_.join(timeout=5)
    print(mode, sorted(res))
