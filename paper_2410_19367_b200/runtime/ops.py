"""Tensor-level wrappers over the C ABI (one call = one library entry point).

Tensors are torch CUDA tensors used purely as device buffers: the wrappers
read ``data_ptr()``/shape/stride, check them, and hand raw pointers plus the
CUDA stream handle to ``libbitpipe_b200.so``.  No computation happens in
torch here.
"""
from __future__ import annotations

import ctypes

import torch

from .lib import (BP_BF16, BP_F32, EPI_DGELU, EPI_GELU, EPI_NONE, GemmArgs, check, lib)

__all__ = ["gemm", "layernorm_fwd", "layernorm_bwd", "colsum_acc", "embed_fwd", "embed_bwd", "xent_fwd_bwd",
           "cast", "attn_fwd", "attn_bwd", "attn_workspace_numel", "adam", "set_option", "launch_count",
           "EPI_NONE", "EPI_GELU", "EPI_DGELU"]


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return BP_F32
    if t.dtype == torch.bfloat16:
        return BP_BF16
    raise TypeError(f"unsupported dtype {t.dtype}")


def _p(t):
    """Device pointer of a tensor, or a raw address (an imported peer buffer)."""
    if t is None:
        return None
    return ctypes.c_void_p(t if isinstance(t, int) else t.data_ptr())


def _s(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _rowmajor(t: torch.Tensor, name: str) -> None:
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError(f"{name} must be a 2-D row-major view (stride(1)==1), got {tuple(t.stride())}")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")


# Optional live probe of the tensor-core GEMM launches (bench.py): CUDA
# events recorded on the launching stream around every bf16 bp_gemm call.
_gemm_probe = None


def gemm_probe_start() -> None:
    global _gemm_probe
    _gemm_probe = []


def gemm_probe_stop():
    """Returns [(flops, shape, start_event, end_event)] of the probed launches."""
    global _gemm_probe
    out, _gemm_probe = _gemm_probe, None
    return out or []


def set_option(option: int, value: int) -> None:
    check(lib().bp_set_option(option, int(value)), "bp_set_option")


def launch_count() -> int:
    return int(lib().bp_launch_count())


def gemm(a, b, c, *, a_kmajor=True, b_kmajor=True, alpha=1.0, beta=0.0, bias=None, residual=None, aux=None,
         epilogue=EPI_NONE, stream=None, force_simt=False, colsum=None):
    """c = epilogue(alpha * op(a) @ op(b)); see include/bitpipe.h for op().
    colsum (fp32 [N]): += column sums of c as stored (fused bias gradient)."""
    for t, n in ((a, "a"), (b, "b"), (c, "c")):
        _rowmajor(t, n)
    M, K = (a.shape if a_kmajor else (a.shape[1], a.shape[0]))
    N, K2 = (b.shape if b_kmajor else (b.shape[1], b.shape[0]))
    if K != K2 or tuple(c.shape) != (M, N):
        raise ValueError(f"gemm shape mismatch: op(a)={M}x{K} op(b)={K2}x{N} c={tuple(c.shape)}")
    if a.dtype != b.dtype:
        raise TypeError("gemm operands must share a dtype")
    g = GemmArgs()
    g.M, g.N, g.K = int(M), int(N), int(K)
    g.in_dtype = _dt(a)
    g.a_kmajor, g.b_kmajor = int(bool(a_kmajor)), int(bool(b_kmajor))
    g.A, g.lda = a.data_ptr(), a.stride(0)
    g.B, g.ldb = b.data_ptr(), b.stride(0)
    g.C, g.ldc, g.c_dtype = c.data_ptr(), c.stride(0), _dt(c)
    g.alpha, g.beta = float(alpha), float(beta)
    g.bias = bias.data_ptr() if bias is not None else None
    if residual is not None:
        _rowmajor(residual, "residual")
        g.residual, g.ldr = residual.data_ptr(), residual.stride(0)
    if aux is not None:
        _rowmajor(aux, "aux")
        g.aux, g.ldaux = aux.data_ptr(), aux.stride(0)
    g.epilogue = int(epilogue)
    g.force_simt = int(bool(force_simt))
    if colsum is not None:
        if colsum.dtype != torch.float32 or colsum.numel() != N:
            raise ValueError("colsum must be an fp32 [N] tensor")
        g.colsum = colsum.data_ptr()
    probe = _gemm_probe is not None and g.in_dtype == BP_BF16
    if probe:
        st = stream if stream is not None else torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
    check(lib().bp_gemm(ctypes.byref(g), _s(stream)), "bp_gemm")
    if probe:
        e1.record(st)
        _gemm_probe.append((2.0 * M * N * K, (int(M), int(N), int(K)), e0, e1))


def layernorm_fwd(x, gamma, beta, y, mean, rstd, eps=1e-5, stream=None):
    rows, cols = x.shape
    check(lib().bp_layernorm_fwd(_dt(x), rows, cols, _p(x), _p(gamma), _p(beta), float(eps), _p(y), _p(mean),
                                 _p(rstd), _s(stream)), "bp_layernorm_fwd")


def layernorm_bwd(dy, x, gamma, mean, rstd, dx, dgamma, dbeta, dres=None, dx_colsum=None, stream=None):
    """dx = dres + dLN(dy); dgamma/dbeta (+ dx_colsum, the column sum of dx) accumulate in fp32."""
    rows, cols = x.shape
    check(lib().bp_layernorm_bwd_ex(_dt(x), rows, cols, _p(dy), _p(x), _p(gamma), _p(mean), _p(rstd), _p(dres),
                                    _p(dx), _p(dgamma), _p(dbeta), _p(dx_colsum), _s(stream)), "bp_layernorm_bwd")


def colsum_acc(x, out, stream=None):
    _rowmajor(x, "x")
    rows, cols = x.shape
    check(lib().bp_colsum_acc(_dt(x), rows, cols, _p(x), x.stride(0), _p(out), _s(stream)), "bp_colsum_acc")


def embed_fwd(tokens, wte, wpe, out, B, S, stream=None):
    H = wte.shape[1]
    check(lib().bp_embed_fwd(_dt(wte), B, S, H, _p(tokens), _p(wte), _p(wpe), _p(out), _s(stream)), "bp_embed_fwd")


def embed_bwd(tokens, dout, dwte, dwpe, B, S, stream=None):
    H = dout.shape[1]
    check(lib().bp_embed_bwd(_dt(dout), B, S, H, _p(tokens), _p(dout), _p(dwte), _p(dwpe), _s(stream)),
          "bp_embed_bwd")


def xent_fwd_bwd(logits, targets, loss_out, grad_scale, loss_scale, stream=None):
    _rowmajor(logits, "logits")
    rows, V = logits.shape
    check(lib().bp_xent_fwd_bwd(_dt(logits), rows, V, _p(logits), logits.stride(0), _p(targets),
                                float(grad_scale), float(loss_scale), _p(loss_out), _s(stream)), "bp_xent_fwd_bwd")


def cast(src, dst, stream=None):
    check(lib().bp_cast(_dt(src), _dt(dst), src.numel(), _p(src), _p(dst), _s(stream)), "bp_cast")


def attn_workspace_numel(B, S, H, Dh) -> int:
    return int(lib().bp_attn_workspace_bytes(B, S, H, Dh)) // 4


def attn_fwd(qkv, o, lse, B, S, H, Dh, causal, scale, stream=None):
    check(lib().bp_attn_fwd(_dt(qkv), B, S, H, Dh, int(bool(causal)), float(scale), _p(qkv), _p(o), _p(lse),
                            _s(stream)), "bp_attn_fwd")


def attn_bwd(qkv, o, dout, lse, dqkv, workspace, B, S, H, Dh, causal, scale, stream=None, dbias=None):
    """dqkv = attention backward; dbias (fp32 [3*H*Dh]) += column sums of dqkv
    (the QKV bias gradient, fused into the tcgen05 kernels)."""
    if dbias is not None and (dbias.dtype != torch.float32 or dbias.numel() != 3 * H * Dh):
        raise ValueError("dbias must be an fp32 [3*H*Dh] tensor")
    need = attn_workspace_numel(B, S, H, Dh)
    if workspace.dtype != torch.float32 or workspace.numel() < need:
        raise ValueError(f"attention workspace must be fp32 with >= {need} elements (attn_workspace_numel)")
    check(lib().bp_attn_bwd_ex(_dt(qkv), B, S, H, Dh, int(bool(causal)), float(scale), _p(qkv), _p(o), _p(dout),
                               _p(lse), _p(dqkv), _p(workspace), _p(dbias), _s(stream)), "bp_attn_bwd")


def adam(master, grad_a, grad_b, m, v, param_a, param_b, *, lr, beta1, beta2, eps, weight_decay, step,
         grad_scale=1.0, stream=None, step_dev=None):
    """Fused replica-mean AdamW; ``step_dev`` (int32 device scalar) makes the
    kernel read the step on the device (CUDA-graph capturable)."""
    pdt = _dt(param_a) if param_a is not None else BP_F32
    check(lib().bp_adam_dev(master.numel(), pdt, _p(master), _p(grad_a), _p(grad_b), _p(m), _p(v), _p(param_a),
                            _p(param_b), float(lr), float(beta1), float(beta2), float(eps), float(weight_decay),
                            int(step), _p(step_dev), float(grad_scale), _s(stream)), "bp_adam")
