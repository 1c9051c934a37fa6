"""One virtual stage's forward / backward pass as a sequence of C-ABI kernels.

This is the body of the reference SPEC's per-task work ("each
worker executes its task list in order; activations/gradients flow along
schedule edges; gradients accumulate over micro-batches") for the
transformer stages of ``model.py``.  Every launch goes to
``libbitpipe_b200.so`` on the logical device's stream; torch only provides
the buffers.

Per half-block (x = residual stream, M = B*S tokens):
  attn fwd : a=LN1(x) | qkv=a W^T+b (tcgen05) | o=attn(qkv) | x'=x+o Wo^T+bo
             (bias + residual fused in the GEMM epilogue)
  mlp  fwd : m=LN2(x) | g=gelu(m W1^T+b1), u saved (GELU epilogue) |
             x'=x+g W2^T+b2
  attn bwd : dWo+=dy^T o | dbo+=sum dy | do=dy Wo | dqkv=attn_bwd (+dbqkv
             in its epilogues) | dWqkv+=dqkv^T a | da=dqkv Wqkv |
             dx=dy+LN1'(da)
  mlp  bwd : dW2+=dy^T g | db2 | du=(dy W2)*gelu'(u) (dGELU epilogue, +db1
             column sums) | dW1+=du^T m | dm=du W1 | dx=dy+LN2'(dm)
  head     : xf=LNf(x) | logits=xf Wlm^T | fused softmax-CE fwd+bwd in place
             (loss to the micro-batch's slot) ; bwd: dxf=dlogits Wlm,
             dWlm+=dlogits^T xf, dx=LNf'(dxf)
  embed    : x0=wte[tok]+wpe ; bwd: scatter-add into dwte, dwpe
Weight gradients accumulate in fp32 directly in the GEMM epilogue (beta=1).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

from ..model import ModelConfig, StagePlan
from . import ops
from .lib import EPI_DGELU, EPI_GELU
from .state import BufferPool, StageParams

__all__ = ["Stash", "StageCompute"]


@dataclass
class Stash:
    xs: list                      # residual stream: xs[0] = stage input
    saves: list = field(default_factory=list)
    head: tuple | None = None
    tokens: torch.Tensor | None = None
    slot: int = 0                 # micro-batch slot of this iteration (deferred weight gradients)
    pinned: set = field(default_factory=set)  # ids of slot views: never released to the pool

    def buffers(self):
        out = list(self.xs)
        for s in self.saves:
            out.extend(s[1:])
        if self.head is not None:
            out.extend(self.head)
        return [t for t in out if id(t) not in self.pinned]


class StageCompute:
    """Forward/backward of one stage replica with a fixed parameter store."""

    def __init__(self, cfg: ModelConfig, plan: StagePlan, params: StageParams, *, grad_scale: float,
                 n_rep: int = 1, defer_wgrad: bool = True):
        self.cfg, self.plan, self.sp = cfg, plan, params
        self.dtype = params.dtype
        self.M = cfg.micro_batch * cfg.seq
        self.grad_scale = grad_scale          # d(step objective)/d(micro-batch mean loss)
        self.loss_scale = 1.0 / self.M
        self.wgrad_beta = 1.0                 # 0.0 for the first backward of an iteration
        # Deferred weight gradients: the weight-gradient GEMM operands of the
        # replica's n_rep micro-batches (LN outputs, attention / GELU outputs,
        # output gradients, dQKV, dU, LN-f output, dlogits) are written into
        # per-iteration slots [n_rep * M, width]; the replica's last backward
        # of the iteration issues ONE GEMM per weight over all of them
        # (K = n_rep M, beta = 0): dW is written once instead of n_rep fp32
        # read-modify-write passes, and the GEMMs are 8x deeper.
        self.n_rep = n_rep
        self.defer_wgrad = defer_wgrad and n_rep > 1
        self._slots: dict = {}
        self._fwd_slot = self._bwd_count = 0
        # co-resident bidirectional pipelines: both replicas of a stage share
        # one slot set ([slot_total * M] rows, this replica's micro-batches at
        # rows slot_base * M ...) and the executor issues ONE deferred GEMM per
        # weight over both (K = N M, ``combined_wgrad``): dW is written once
        # per stage and AdamW reads a single gradient for the GEMM weights
        self.slot_base, self.slot_total = 0, n_rep
        self.combined_wgrad = False
        # cross-stage bias-gradient fusion (coresident executor): the output
        # gradient of this stage IS the dx of the next stage's last LayerNorm
        # backward, which accumulates its column sums into this stage's last
        # output-projection bias gradient (``prev_out_bias`` of the next stage)
        self.prev_out_bias = None
        self.out_bias_by_next = False

    def begin_iteration(self):
        """The next backward is this replica's first of the iteration: its
        weight-gradient GEMMs write (beta = 0) instead of accumulating, which
        replaces zeroing the (large) GEMM-weight part of the gradient buffer.
        All backwards of one replica run on one stream, in issue order."""
        self.wgrad_beta = 0.0
        self._fwd_slot = self._bwd_count = 0

    def _slot_all(self, key, width):
        t = self._slots.get(key)
        if t is None:
            t = torch.empty(self.slot_total * self.M, width, dtype=self.dtype, device=self.sp.flat.device)
            self._slots[key] = t
        return t

    def _buf(self, st: Stash, key, width, pool, stream):
        """This micro-batch's slot view of ``key`` (deferred mode, pinned in
        the stash) or a pool buffer."""
        if not self.defer_wgrad:
            return pool.get((self.M, width), self.dtype, stream)
        M, k = self.M, self.slot_base + st.slot
        t = self._slot_all(key, width)[k * M:(k + 1) * M]
        st.pinned.add(id(t))
        return t

    # ------------------------------------------------------------- forward --
    def forward(self, stream, pool: BufferPool, *, x0=None, tokens=None, targets=None, loss_slot=None):
        cfg, P = self.cfg, self.sp.p
        M, h, dt = self.M, cfg.hidden, self.dtype
        f32 = torch.float32
        if self.plan.embed:
            x0 = pool.get((M, h), dt, stream)
            ops.embed_fwd(tokens, P["embed.wte"], P["embed.wpe"], x0, cfg.micro_batch, cfg.seq, stream=stream)
        st = Stash(xs=[x0], tokens=tokens)
        if self.defer_wgrad:
            st.slot = self._fwd_slot % self.n_rep
            self._fwd_slot += 1
        H, Dh = cfg.heads, cfg.head_dim
        scale = 1.0 / math.sqrt(Dh)
        for hb in self.plan.halfblocks:
            l, half = divmod(hb, 2)
            p = f"layers.{l}."
            x = st.xs[-1]
            mean, rstd = pool.get((M,), f32, stream), pool.get((M,), f32, stream)
            y = pool.get((M, h), dt, stream)
            if half == 0:
                a = self._buf(st, ("a", hb), h, pool, stream)
                ops.layernorm_fwd(x, P[p + "ln1.w"], P[p + "ln1.b"], a, mean, rstd, cfg.ln_eps, stream=stream)
                qkv = pool.get((M, 3 * h), dt, stream)
                ops.gemm(a, P[p + "attn.qkv.w"], qkv, bias=P[p + "attn.qkv.b"], stream=stream)
                o = self._buf(st, ("o", hb), h, pool, stream)
                lse = pool.get((cfg.micro_batch * H * cfg.seq,), f32, stream)
                ops.attn_fwd(qkv, o, lse, cfg.micro_batch, cfg.seq, H, Dh, cfg.causal, scale, stream=stream)
                ops.gemm(o, P[p + "attn.proj.w"], y, bias=P[p + "attn.proj.b"], residual=x, stream=stream)
                st.saves.append(("attn", a, mean, rstd, qkv, o, lse))
            else:
                m = self._buf(st, ("m", hb), h, pool, stream)
                ops.layernorm_fwd(x, P[p + "ln2.w"], P[p + "ln2.b"], m, mean, rstd, cfg.ln_eps, stream=stream)
                u = pool.get((M, cfg.ffn), dt, stream)
                g = self._buf(st, ("g", hb), cfg.ffn, pool, stream)
                ops.gemm(m, P[p + "mlp.fc1.w"], g, bias=P[p + "mlp.fc1.b"], aux=u, epilogue=EPI_GELU, stream=stream)
                ops.gemm(g, P[p + "mlp.fc2.w"], y, bias=P[p + "mlp.fc2.b"], residual=x, stream=stream)
                st.saves.append(("mlp", m, mean, rstd, u, g))
            st.xs.append(y)
        if self.plan.head:
            x = st.xs[-1]
            xf = self._buf(st, ("xf",), h, pool, stream)
            mean, rstd = pool.get((M,), f32, stream), pool.get((M,), f32, stream)
            ops.layernorm_fwd(x, P["head.lnf.w"], P["head.lnf.b"], xf, mean, rstd, cfg.ln_eps, stream=stream)
            logits = self._buf(st, ("logits",), cfg.vocab, pool, stream)
            ops.gemm(xf, P["head.lm.w"], logits, stream=stream)
            ops.xent_fwd_bwd(logits, targets, loss_slot, grad_scale=self.grad_scale * self.loss_scale,
                             loss_scale=self.loss_scale, stream=stream)
            st.head = (xf, mean, rstd, logits)
            return st, None
        out = st.xs.pop()          # ownership moves to the consumer of the message
        return st, out

    # ------------------------------------------------------------ backward --
    def _out_bias_grad(self, i):
        """fp32 gradient of the output-projection bias of local half-block i
        (None when i < 0): the column sum of that half-block's output grad."""
        if i < 0:
            return None
        l, half = divmod(self.plan.halfblocks[i], 2)
        return self.sp.g[f"layers.{l}." + ("attn.proj.b" if half == 0 else "mlp.fc2.b")]

    @staticmethod
    def _wgrad(stream, wstream, fn):
        """Issue weight-gradient GEMMs: on ``stream``, or (``wstream``) on the
        side stream behind everything ``stream`` has issued so far, so they
        overlap the rest of the task's input-gradient chain (which carries
        the pipeline's critical path to the previous stage)."""
        if wstream is None:
            fn(stream)
            return
        ev = torch.cuda.Event()
        ev.record(stream)
        wstream.wait_event(ev)
        fn(wstream)

    def _deferred_wgrads(self, q, rows=None):
        """All of the iteration's weight gradients of this replica (or, with
        shared slots, of both co-resident replicas), one GEMM per weight over
        the slot_total micro-batch slots (beta = 0).  ``rows`` = (r0, r1)
        restricts K to those slot rows (one replica's share, for timing)."""
        G, S = self.sp.g, self._slots
        if rows is not None:
            S = {k: v[rows[0]:rows[1]] for k, v in S.items()}
        for hb in self.plan.halfblocks:
            l, half = divmod(hb, 2)
            p = f"layers.{l}."
            if half == 0:
                ops.gemm(S[("dy", hb)], S[("o", hb)], G[p + "attn.proj.w"], a_kmajor=False, b_kmajor=False,
                         beta=0.0, stream=q)
                ops.gemm(S[("dqkv", hb)], S[("a", hb)], G[p + "attn.qkv.w"], a_kmajor=False, b_kmajor=False,
                         beta=0.0, stream=q)
            else:
                ops.gemm(S[("dy", hb)], S[("g", hb)], G[p + "mlp.fc2.w"], a_kmajor=False, b_kmajor=False,
                         beta=0.0, stream=q)
                ops.gemm(S[("du", hb)], S[("m", hb)], G[p + "mlp.fc1.w"], a_kmajor=False, b_kmajor=False,
                         beta=0.0, stream=q)
        if self.plan.head:
            ops.gemm(S[("logits",)], S[("xf",)], G["head.lm.w"], a_kmajor=False, b_kmajor=False, beta=0.0,
                     stream=q)

    def backward(self, stream, pool: BufferPool, st: Stash, dy, ws, wstream=None, dx_dest=None):
        """Returns (dx0 or None, buffers to release after the task's ``stream``
        work, buffers also read by side-stream weight-gradient GEMMs).
        ``dx_dest``: where to write the input gradient (the message), e.g.
        the previous stage's output-gradient slot; else a pool buffer."""
        cfg, P, G = self.cfg, self.sp.p, self.sp.g
        M, h, dt = self.M, cfg.hidden, self.dtype
        H, Dh = cfg.heads, cfg.head_dim
        scale = 1.0 / math.sqrt(Dh)
        defer = self.defer_wgrad
        release = st.buffers()
        wread = []
        wg = self._wgrad
        wb, self.wgrad_beta = self.wgrad_beta, 1.0
        hbs = self.plan.halfblocks
        nhb = len(hbs)
        if self.plan.head:
            xf, mean, rstd, dlogits = st.head
            dxf = pool.get((M, h), dt, stream)
            ops.gemm(dlogits, P["head.lm.w"], dxf, b_kmajor=False, stream=stream)
            if not defer:
                wg(stream, wstream, lambda q: ops.gemm(dlogits, xf, G["head.lm.w"], a_kmajor=False, b_kmajor=False,
                                                       beta=wb, stream=q))
                wread += [dlogits, xf]
            # gradient w.r.t. the last half-block's output (a wgrad operand
            # slot), or the message when the stage has no half-block
            dy = self._buf(st, ("dy", hbs[-1]), h, pool, stream) if nhb else \
                (dx_dest if dx_dest is not None else pool.get((M, h), dt, stream))
            # the LN backward also sums its dx over rows: that is the output-bias
            # gradient of the half-block before it (fused, no separate launch)
            ops.layernorm_bwd(dxf, st.xs[-1], P["head.lnf.w"], mean, rstd, dy, G["head.lnf.w"], G["head.lnf.b"],
                              dx_colsum=self._out_bias_grad(nhb - 1) if nhb else self.prev_out_bias, stream=stream)
            bias_done = bool(nhb)
            release += [dxf, dy]
        else:
            release.append(dy)
            if defer and nhb:  # the incoming message into this micro-batch's output-gradient slot
                dys = self._buf(st, ("dy", hbs[-1]), h, pool, stream)
                if dys.data_ptr() != dy.data_ptr():   # (the co-resident producer wrote it there already)
                    with torch.cuda.stream(stream):
                        dys.copy_(dy)
                dy = dys
            bias_done = self.out_bias_by_next
        for i in range(nhb - 1, -1, -1):
            l, half = divmod(hbs[i], 2)
            p = f"layers.{l}."
            x = st.xs[i]
            save = st.saves[i]
            # gradient w.r.t. this half-block's input = the previous half-block's output gradient
            dx = self._buf(st, ("dy", hbs[i - 1]), h, pool, stream) if i > 0 else \
                (dx_dest if dx_dest is not None and not self.plan.embed else pool.get((M, h), dt, stream))
            if half == 0:
                _, a, mean, rstd, qkv, o, lse = save
                if not defer:
                    wg(stream, wstream, lambda q: ops.gemm(dy, o, G[p + "attn.proj.w"], a_kmajor=False,
                                                           b_kmajor=False, beta=wb, stream=q))
                    wread += [dy, o]
                if not bias_done:
                    ops.colsum_acc(dy, G[p + "attn.proj.b"], stream=stream)
                do = pool.get((M, h), dt, stream)
                ops.gemm(dy, P[p + "attn.proj.w"], do, b_kmajor=False, stream=stream)
                dqkv = self._buf(st, ("dqkv", hbs[i]), 3 * h, pool, stream)
                # the QKV bias gradient (column sums of dqkv) comes out of the
                # attention backward's epilogues
                ops.attn_bwd(qkv, o, do, lse, dqkv, ws, cfg.micro_batch, cfg.seq, H, Dh, cfg.causal, scale,
                             stream=stream, dbias=G[p + "attn.qkv.b"])
                if not defer:
                    wg(stream, wstream, lambda q: ops.gemm(dqkv, a, G[p + "attn.qkv.w"], a_kmajor=False,
                                                           b_kmajor=False, beta=wb, stream=q))
                    wread += [dqkv, a]
                da = pool.get((M, h), dt, stream)
                ops.gemm(dqkv, P[p + "attn.qkv.w"], da, b_kmajor=False, stream=stream)
                ops.layernorm_bwd(da, x, P[p + "ln1.w"], mean, rstd, dx, G[p + "ln1.w"], G[p + "ln1.b"], dres=dy,
                                  dx_colsum=self._out_bias_grad(i - 1) if i else self.prev_out_bias, stream=stream)
                release += [do, dqkv, da]
            else:
                _, m, mean, rstd, u, g = save
                if not defer:
                    wg(stream, wstream, lambda q: ops.gemm(dy, g, G[p + "mlp.fc2.w"], a_kmajor=False,
                                                           b_kmajor=False, beta=wb, stream=q))
                    wread += [dy, g]
                if not bias_done:
                    ops.colsum_acc(dy, G[p + "mlp.fc2.b"], stream=stream)
                du = self._buf(st, ("du", hbs[i]), cfg.ffn, pool, stream)
                # du = (dy W2) * gelu'(u); its column sums (the fc1 bias
                # gradient) are reduced in the same GEMM epilogue
                ops.gemm(dy, P[p + "mlp.fc2.w"], du, b_kmajor=False, aux=u, epilogue=EPI_DGELU, stream=stream,
                         colsum=G[p + "mlp.fc1.b"])
                if not defer:
                    wg(stream, wstream, lambda q: ops.gemm(du, m, G[p + "mlp.fc1.w"], a_kmajor=False,
                                                           b_kmajor=False, beta=wb, stream=q))
                    wread += [du, m]
                dm = pool.get((M, h), dt, stream)
                ops.gemm(du, P[p + "mlp.fc1.w"], dm, b_kmajor=False, stream=stream)
                ops.layernorm_bwd(dm, x, P[p + "ln2.w"], mean, rstd, dx, G[p + "ln2.w"], G[p + "ln2.b"], dres=dy,
                                  dx_colsum=self._out_bias_grad(i - 1) if i else self.prev_out_bias, stream=stream)
                release += [du, dm]
            if i > 0 or self.plan.embed:
                release.append(dx)
            bias_done = i > 0
            dy = dx
        if defer:
            self._bwd_count += 1
            if self._bwd_count == self.n_rep and not self.combined_wgrad:  # every micro-batch is in the slots
                wg(stream, wstream, self._deferred_wgrads)
        if self.plan.embed:
            ops.embed_bwd(st.tokens, dy, G["embed.wte"], G["embed.wpe"], cfg.micro_batch, cfg.seq, stream=stream)
            dx0 = None
        else:  # dy is now the gradient w.r.t. the stage input: it becomes the message
            dx0 = dy
            release = [t for t in release if t is not dy]
        release = [t for t in release if id(t) not in st.pinned]
        if wstream is None or defer:
            return dx0, release, []
        wids = {id(t) for t in wread}
        return dx0, [t for t in release if id(t) not in wids], [t for t in release if id(t) in wids]
