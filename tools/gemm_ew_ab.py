"""A/B of the 2-SM GEMM's epilogue warp count (BP_OPT_GEMM_EPI_WARPS 4 vs 8)
on the per-micro-batch shapes of the GPT-1.3B / BERT-large / GPT-10B steps
with the epilogues the executor uses (bias, bias + residual, GELU, dGELU,
column sums).  Checks both variants produce the same bytes, then times them
interleaved (clock drift hits both alike).  `python tools/gemm_ew_ab.py`."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_19367_b200.runtime import lib as L
from paper_2410_19367_b200.runtime import ops


def timeit(fn, iters=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / iters


def case(name, M, N, K, epi, ak=True, bk=True):
    dev = "cuda"
    A = (torch.randn(M, K, device=dev) if ak else torch.randn(K, M, device=dev)).bfloat16()
    B = (torch.randn(N, K, device=dev) if bk else torch.randn(K, N, device=dev)).bfloat16() * 0.02
    C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    kw = {}
    if "bias" in epi:
        kw["bias"] = torch.randn(N, device=dev).bfloat16()  # the bias has the operands' dtype
    if "res" in epi:
        kw["residual"] = torch.randn(M, N, device=dev).bfloat16()
    if "gelu" in epi:
        kw["aux"] = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        kw["epilogue"] = L.EPI_GELU
    if "dgelu" in epi:
        kw["aux"] = torch.randn(M, N, device=dev).bfloat16()
        kw["epilogue"] = L.EPI_DGELU
    if "colsum" in epi:
        kw["colsum"] = torch.zeros(N, device=dev)

    def run():
        if "colsum" in kw:
            kw["colsum"].zero_()
        ops.gemm(A, B, C, a_kmajor=ak, b_kmajor=bk, **kw)

    outs = {}
    for ew in (4, 8):
        ops.set_option(L.OPT_GEMM_EPI_WARPS, ew)
        run()
        torch.cuda.synchronize()
        outs[ew] = C.clone(), (kw["aux"].clone() if kw.get("epilogue") == L.EPI_GELU else None)
    bits = lambda t: t.view(torch.int16)  # bit patterns: NaN-safe
    same = torch.equal(bits(outs[4][0]), bits(outs[8][0])) and (
        outs[4][1] is None or torch.equal(bits(outs[4][1]), bits(outs[8][1])))
    if not same:
        d = (outs[4][0].float() - outs[8][0].float()).abs()
        bad = (bits(outs[4][0]) != bits(outs[8][0])).nonzero()
        print(f"  DIFF {name}: {bad.shape[0]} elements, max {d.max().item():.3g}, rows {bad[:, 0].unique()[:8].tolist()} "
              f"cols {bad[:, 1].unique()[:16].tolist()}", flush=True)
    t = {4: [], 8: []}
    for _ in range(3):
        for ew in (4, 8):
            ops.set_option(L.OPT_GEMM_EPI_WARPS, ew)
            t[ew].append(timeit(run))
    t4, t8 = min(t[4]), min(t[8])
    fl = 2.0 * M * N * K
    print(f"{name:28s} {M:6d}x{N:6d}x{K:6d} {epi:12s} ew4 {t4:7.1f} us ({fl / t4 / 1e6:6.0f} TF/s)  "
          f"ew8 {t8:7.1f} us ({fl / t8 / 1e6:6.0f} TF/s)  x{t4 / t8:.3f}  {'same' if same else 'DIFF'}", flush=True)
    ops.set_option(L.OPT_GEMM_EPI_WARPS, 0)
    return same


T = 2048
ok = True
if len(sys.argv) > 1:  # quick check: the first case only, three times
    for _ in range(3):
        case("gpt-1.3b qkv fprop", T, 3 * 2048, 2048, "bias")
    sys.exit(0)
for h, f, tag in ((2048, 8192, "gpt-1.3b"), (1024, 4096, "bert-large"), (4096, 16384, "gpt-10b")):
    ok &= case(f"{tag} qkv fprop", T, 3 * h, h, "bias")
    ok &= case(f"{tag} proj fprop", T, h, h, "bias+res")
    ok &= case(f"{tag} fc1 fprop", T, f, h, "bias+gelu")
    ok &= case(f"{tag} fc2 fprop", T, h, f, "bias+res")
    ok &= case(f"{tag} fc2 dgrad", T, f, h, "dgelu", bk=False)
    ok &= case(f"{tag} fc1 dgrad", T, h, f, "none", bk=False)
    ok &= case(f"{tag} qkv dgrad", T, h, 3 * h, "none", bk=False)
    ok &= case(f"{tag} proj dgrad", T, h, h, "none", bk=False)
print("all identical" if ok else "MISMATCH")
