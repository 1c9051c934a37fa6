"""Warm-L2 timings of the LayerNorm / column-reduction kernels at GPT-1.3B
shapes (2048 x 2048 bf16) vs a device copy of the same bytes."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import ops
from paper_2410_19367_b200.runtime.lib import OPT_LN_BWD_MODE, OPT_LN_UNFUSED


def timeit(fn, iters=20):
    """Device time per call: `iters` calls captured in one CUDA graph (the
    ctypes launch path costs ~10 us of host time per call, more than these
    kernels take on the device)."""
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / (5 * iters) * 1e3


rows = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
for cols in (2048, 4096):
    x = torch.randn(rows, cols, device="cuda").bfloat16()
    g = torch.randn(cols, device="cuda").bfloat16()
    b = torch.randn(cols, device="cuda").bfloat16()
    y = torch.empty_like(x)
    mean = torch.empty(rows, device="cuda")
    rstd = torch.empty(rows, device="cuda")
    dy, dres, dx = torch.randn_like(x), torch.randn_like(x), torch.empty_like(x)
    dg, db, cs = (torch.zeros(cols, device="cuda") for _ in range(3))
    MB = x.numel() * 2 / 1e6
    t_copy = timeit(lambda: y.copy_(x))
    t_fwd = timeit(lambda: ops.layernorm_fwd(x, g, b, y, mean, rstd))
    ops.set_option(OPT_LN_UNFUSED, 0)
    ops.set_option(OPT_LN_BWD_MODE, 1)
    t_tma = timeit(lambda: ops.layernorm_bwd(dy, x, g, mean, rstd, dx, dg, db, dres=dres, dx_colsum=cs))
    ops.set_option(OPT_LN_BWD_MODE, 0)
    t_bf = timeit(lambda: ops.layernorm_bwd(dy, x, g, mean, rstd, dx, dg, db, dres=dres, dx_colsum=cs))
    t_bf0 = timeit(lambda: ops.layernorm_bwd(dy, x, g, mean, rstd, dx, dg, db, dres=dres))
    ops.set_option(OPT_LN_UNFUSED, 1)
    t_bu = timeit(lambda: ops.layernorm_bwd(dy, x, g, mean, rstd, dx, dg, db, dres=dres, dx_colsum=cs))
    t_bu0 = timeit(lambda: ops.layernorm_bwd(dy, x, g, mean, rstd, dx, dg, db, dres=dres))
    ops.set_option(OPT_LN_UNFUSED, 0)
    cps = []
    for c in (1, 2, 3, 4):
        ops.set_option(9, c)
        cps.append(timeit(lambda: ops.layernorm_bwd(dy, x, g, mean, rstd, dx, dg, db, dres=dres, dx_colsum=cs)))
    ops.set_option(9, 1)
    print("fused ln_bwd by CTAs/SM 1..4:", " ".join(f"{t:.1f}" for t in cps))
    t_cs = timeit(lambda: ops.colsum_acc(dy, cs))
    wide = torch.randn(rows, 4 * cols, device="cuda").bfloat16()
    cs4 = torch.zeros(4 * cols, device="cuda")
    t_cs4 = timeit(lambda: ops.colsum_acc(wide, cs4))
    print(f"ln_bwd single-pass TMA {t_tma:.1f} us vs two-pass {t_bf:.1f} us; colsum {rows}x{4*cols} {t_cs4:.1f} us")
    print(f"{rows}x{cols} ({MB:.0f} MB/matrix): copy {t_copy:.1f} us ({2*MB/t_copy:.2f} TB/s) | ln_fwd {t_fwd:.1f} | "
          f"ln_bwd fused {t_bf:.1f} (no colsum {t_bf0:.1f}) | unfused {t_bu:.1f} (no colsum {t_bu0:.1f}) | "
          f"colsum {t_cs:.1f} us", flush=True)
