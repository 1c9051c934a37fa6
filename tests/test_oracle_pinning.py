"""Pinning the CPU oracle itself (no GPU).

The reference pins no numeric values (it has no train step),
so the oracle is pinned three independent ways:

1. the SPEC ``runtime`` module's own known answers on its ToyModel
   (SPEC.md:426-444), run through the SAME message-passing executor the GPT
   oracle uses (``gpt_oracle.execute_orders``);
2. every piece of the restated transformer against an independent
   implementation in float64: ``torch.nn.functional`` (layer_norm,
   gelu(tanh), scaled_dot_product_attention, cross_entropy),
   ``torch.nn.TransformerEncoderLayer`` (pre-LN, causal and bidirectional)
   and, for the whole causal model, HuggingFace ``GPT2LMHeadModel``
   (loss AND every parameter gradient);
3. the single AdamW update against ``torch.optim.AdamW``.
"""

import pytest
import torch
import torch.nn.functional as F

from oracle import gpt_oracle as go
from oracle.toy_model import ToyModel, toy_run_schedule_numeric, toy_sequential_baseline
from paper_2410_19367_b200 import schedule as ps
from paper_2410_19367_b200.model import CONFIGS, init_params, synthetic_batch



@pytest.fixture(autouse=True)
def _float64_default():
    """float64 tensors by default inside THIS module only (a module-level
    set_default_dtype would leak into every test collected after it)."""
    old = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    yield
    torch.set_default_dtype(old)


def rel(a, b):
    return ((a - b).norm() / b.norm().clamp_min(1e-300)).item()


def _ocfg(cfg, **kw):
    return go.OracleConfig(cfg.layers, cfg.hidden, cfg.heads, cfg.seq, cfg.vocab, cfg.micro_batch, cfg.causal, **kw)


# --------------------------------------------------------------------------
# 1. SPEC ToyModel known answers
# --------------------------------------------------------------------------
def _toy_batch(N, B, d_in, d_out, seed):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(N, B, d_in, generator=g, dtype=torch.float64),
            torch.randn(N, B, d_out, generator=g, dtype=torch.float64))


def test_toy_1f1b_identity_closed_form():
    """1F1B D=2, N=2, identity-initialised single-unit layers
    -> the loss (and gradient, update) in closed form."""
    sched = ps.build(ps.ApproachId.DAPPLE_1F1B, 2, 2)
    model = ToyModel.identity(num_stages=2, width=1, lr=0.1)
    x, t = _toy_batch(2, 3, 1, 1, seed=4)
    res = toy_run_schedule_numeric(ps.dump_schedule(sched), model, (x, t))
    # identity network: output = input
    loss = sum(((x[i] - t[i]) ** 2).mean() for i in range(2)) / 2
    assert abs(res.loss - loss.item()) < 1e-15
    # d/dw_s of mean_i mean((x w0 w1 - t)^2) at w = 1: mean_i mean(2 (x - t) x)
    g = sum((2 * (x[i] - t[i]) * x[i]).mean() for i in range(2)) / 2
    for s in range(2):
        assert abs(res.grads[s].item() - g.item()) < 1e-14
        assert abs(res.weights[s].item() - (1 - 0.1 * g.item())) < 1e-14


def test_toy_scalar_mse_derivative():
    """N=1, one stage, scalar model -> gradient = analytic
    derivative of the MSE."""
    model = ToyModel([torch.tensor([[0.7]])], [1, 1], lr=0.5)
    x = torch.tensor([[[1.5]], ]), torch.tensor([[[0.25]]])
    res = toy_sequential_baseline(model, x)
    xv, tv, w = 1.5, 0.25, 0.7
    assert abs(res.loss - (xv * w - tv) ** 2) < 1e-15
    assert abs(res.grads[0].item() - 2 * (xv * w - tv) * xv) < 1e-15
    assert abs(res.weights[0].item() - (w - 0.5 * 2 * (xv * w - tv) * xv)) < 1e-15
    again = toy_sequential_baseline(model, x)        # SPEC.md:441 determinism
    assert again.loss == res.loss and torch.equal(again.grads[0], res.grads[0])


def test_toy_accumulation_is_mean_of_single_microbatches():
    """N=4 -> gradient equals the mean of the 4
    single-micro-batch gradients."""
    model = ToyModel.random([5, 7, 3], seed=2, activation="tanh")
    x, t = _toy_batch(4, 2, 5, 3, seed=9)
    full = toy_sequential_baseline(model, (x, t))
    singles = [toy_sequential_baseline(model, (x[i:i + 1], t[i:i + 1])) for i in range(4)]
    for s in range(2):
        mean = sum(r.grads[s] for r in singles) / 4
        assert rel(full.grads[s], mean) < 1e-13


@pytest.mark.parametrize("approach,D,N", [("bitpipe", 4, 4), ("bitpipe", 2, 4), ("bitpipe", 4, 8),
                                          ("bitpipe-early-forward", 4, 8), ("chimera", 4, 4),
                                          ("dapple-1f1b", 4, 4), ("gpipe", 4, 4), ("interleaved-looping", 4, 8)])
@pytest.mark.parametrize("activation", ["none", "tanh"])
def test_toy_schedule_independence(approach, D, N, activation):
    """run_schedule_numeric == sequential_baseline within
    1e-9 relative (fp64) for every builder; BitPipe D=4 N=4 on an 8-stage
    toy model is the SPEC's own example."""
    sched = ps.build(ps.ApproachId(approach), D, N)
    S = sched.num_stages
    dims = [4 + (s % 3) for s in range(S + 1)]
    model = ToyModel.random(dims, seed=S + N, activation=activation)
    batch = _toy_batch(N, 2, dims[0], dims[-1], seed=D * N)
    run = toy_run_schedule_numeric(ps.dump_schedule(sched), model, batch)
    seq = toy_sequential_baseline(model, batch)
    assert abs(run.loss - seq.loss) <= 1e-12 * abs(seq.loss)
    for s in range(S):
        assert rel(run.grads[s], seq.grads[s]) < 1e-9
        assert rel(run.weights[s], seq.weights[s]) < 1e-12


def test_toy_gpipe_equals_bitpipe():
    """GPipe vs BitPipe on the same model/batch/seed ->
    identical StepResult within 1e-9."""
    model = ToyModel.random([3] * 9, seed=5, activation="tanh")
    batch = _toy_batch(4, 2, 3, 3, seed=6)
    a = toy_run_schedule_numeric(ps.dump_schedule(ps.build(ps.ApproachId.GPIPE, 8, 4)), model, batch)
    b = toy_run_schedule_numeric(ps.dump_schedule(ps.build(ps.ApproachId.BITPIPE, 4, 4)), model, batch)
    assert abs(a.loss - b.loss) < 1e-12
    assert all(rel(x, y) < 1e-9 for x, y in zip(a.grads, b.grads))


def test_toy_shape_mismatch():
    sched = ps.build(ps.ApproachId.BITPIPE, 4, 4)
    with pytest.raises(ValueError, match="ShapeMismatch"):
        toy_run_schedule_numeric(ps.dump_schedule(sched), ToyModel.random([2] * 5), _toy_batch(4, 1, 2, 2, 0))


def test_gpt_oracle_executor_deadlock_detected():
    """A corrupted order (a backward moved before its forward) must abort."""
    import json
    sch = json.loads(ps.dump_schedule(ps.build(ps.ApproachId.BITPIPE, 2, 4)))
    row = sch["per_device"][0]
    row.insert(0, row.pop(next(i for i, r in enumerate(row) if r[0] == "B")))
    model = ToyModel.random([2] * 5, seed=1)
    with pytest.raises(RuntimeError, match="deadlock"):
        toy_run_schedule_numeric(sch, model, _toy_batch(4, 1, 2, 2, 0))


# --------------------------------------------------------------------------
# 2. the restated transformer vs independent implementations (float64)
# --------------------------------------------------------------------------
def _params(cfg, seed=3):
    return {k: v.double() for k, v in init_params(cfg, seed, perturb=True).items()}


def test_layernorm_gelu_match_functional():
    g = torch.Generator().manual_seed(0)
    x = torch.randn(3, 5, 64, generator=g)
    w, b = torch.randn(64, generator=g), torch.randn(64, generator=g)
    assert rel(go._ln(x, w, b, 1e-5), F.layer_norm(x, (64,), w, b, 1e-5)) < 1e-14
    assert rel(go._gelu(x * 4), F.gelu(x * 4, approximate="tanh")) < 1e-15


@pytest.mark.parametrize("causal", [True, False])
def test_halfblocks_match_functional(causal):
    cfg = CONFIGS["tiny"] if causal else CONFIGS["small-bert"]
    oc = _ocfg(cfg)
    P = _params(cfg)
    h, H = cfg.hidden, cfg.heads
    x = torch.randn(cfg.micro_batch, cfg.seq, h, generator=torch.Generator().manual_seed(1))
    p = "layers.0."
    # attention half through F.layer_norm / F.linear / F.scaled_dot_product_attention
    a = F.layer_norm(x, (h,), P[p + "ln1.w"], P[p + "ln1.b"], cfg.ln_eps)
    q, k, v = F.linear(a, P[p + "attn.qkv.w"], P[p + "attn.qkv.b"]).split(h, -1)
    heads = lambda t: t.view(cfg.micro_batch, cfg.seq, H, h // H).transpose(1, 2)  # noqa: E731
    o = F.scaled_dot_product_attention(heads(q), heads(k), heads(v), is_causal=causal)
    ref = x + F.linear(o.transpose(1, 2).reshape_as(x), P[p + "attn.proj.w"], P[p + "attn.proj.b"])
    assert rel(go._attn_half(P, 0, x, oc), ref) < 1e-13
    # MLP half
    m = F.layer_norm(x, (h,), P[p + "ln2.w"], P[p + "ln2.b"], cfg.ln_eps)
    u = F.gelu(F.linear(m, P[p + "mlp.fc1.w"], P[p + "mlp.fc1.b"]), approximate="tanh")
    ref = x + F.linear(u, P[p + "mlp.fc2.w"], P[p + "mlp.fc2.b"])
    assert rel(go._mlp_half(P, 0, x, oc), ref) < 1e-13


@pytest.mark.parametrize("causal", [True, False])
def test_block_matches_transformer_encoder_layer(causal):
    """One pre-LN block (attention half + MLP half) == torch's
    TransformerEncoderLayer(norm_first=True), forward and input gradient."""
    cfg = CONFIGS["tiny"] if causal else CONFIGS["small-bert"]
    oc = _ocfg(cfg)
    P = _params(cfg, seed=5)
    h, p = cfg.hidden, "layers.0."
    layer = torch.nn.TransformerEncoderLayer(h, cfg.heads, dim_feedforward=4 * h, dropout=0.0,
                                             activation=lambda t: F.gelu(t, approximate="tanh"),
                                             layer_norm_eps=cfg.ln_eps, batch_first=True, norm_first=True,
                                             dtype=torch.float64)
    with torch.no_grad():
        sa = layer.self_attn
        sa.in_proj_weight.copy_(P[p + "attn.qkv.w"]); sa.in_proj_bias.copy_(P[p + "attn.qkv.b"])  # noqa: E702
        sa.out_proj.weight.copy_(P[p + "attn.proj.w"]); sa.out_proj.bias.copy_(P[p + "attn.proj.b"])  # noqa: E702
        layer.norm1.weight.copy_(P[p + "ln1.w"]); layer.norm1.bias.copy_(P[p + "ln1.b"])  # noqa: E702
        layer.norm2.weight.copy_(P[p + "ln2.w"]); layer.norm2.bias.copy_(P[p + "ln2.b"])  # noqa: E702
        layer.linear1.weight.copy_(P[p + "mlp.fc1.w"]); layer.linear1.bias.copy_(P[p + "mlp.fc1.b"])  # noqa: E702
        layer.linear2.weight.copy_(P[p + "mlp.fc2.w"]); layer.linear2.bias.copy_(P[p + "mlp.fc2.b"])  # noqa: E702
    layer.train()  # the fast path is inference-only; dropout is 0
    x = torch.randn(cfg.micro_batch, cfg.seq, h, generator=torch.Generator().manual_seed(2), requires_grad=True)
    mask = torch.nn.Transformer.generate_square_subsequent_mask(cfg.seq, dtype=torch.float64) if causal else None
    ref = layer(x, src_mask=mask, is_causal=causal)
    ours = go._mlp_half(P, 0, go._attn_half(P, 0, x, oc), oc)
    assert rel(ours, ref) < 1e-13
    gy = torch.randn_like(ref)
    (gx_ref,) = torch.autograd.grad(ref, x, gy)
    (gx,) = torch.autograd.grad(ours, x, gy)
    assert rel(gx, gx_ref) < 1e-12


def test_head_loss_matches_logsumexp():
    cfg = CONFIGS["tiny"]
    P = _params(cfg)
    g = torch.Generator().manual_seed(3)
    x = torch.randn(cfg.micro_batch, cfg.seq, cfg.hidden, generator=g)
    tgt = torch.randint(0, cfg.vocab, (cfg.micro_batch, cfg.seq), generator=g)
    xf = F.layer_norm(x, (cfg.hidden,), P["head.lnf.w"], P["head.lnf.b"], cfg.ln_eps)
    z = (xf @ P["head.lm.w"].t()).reshape(-1, cfg.vocab)
    ref = (z.logsumexp(-1) - z.gather(1, tgt.reshape(-1, 1)).squeeze(1)).mean()
    assert abs(go._head_loss(P, x, tgt, _ocfg(cfg)).item() - ref.item()) < 1e-13 * ref.item()


def test_whole_gpt_matches_huggingface_gpt2():
    """The oracle's whole causal model (sequential baseline over N
    micro-batches) == HuggingFace GPT2LMHeadModel with the same weights
    (pre-LN, learned positions, gelu_new = tanh-GELU, untied head): loss and
    EVERY parameter gradient, float64."""
    transformers = pytest.importorskip("transformers")
    cfg = CONFIGS["tiny"]
    P = _params(cfg, seed=8)
    N = 2
    tok, tgt = synthetic_batch(cfg, N, seed=4)
    seq = go.sequential_baseline(_ocfg(cfg), P, tok, tgt)

    hc = transformers.GPT2Config(vocab_size=cfg.vocab, n_positions=cfg.seq, n_embd=cfg.hidden, n_layer=cfg.layers,
                                 n_head=cfg.heads, activation_function="gelu_new", layer_norm_epsilon=cfg.ln_eps,
                                 resid_pdrop=0.0, embd_pdrop=0.0, attn_pdrop=0.0, tie_word_embeddings=False)
    hc._attn_implementation = "eager"
    model = transformers.GPT2LMHeadModel(hc).double()
    model.train()
    sd = {"transformer.wte.weight": P["embed.wte"], "transformer.wpe.weight": P["embed.wpe"],
          "transformer.ln_f.weight": P["head.lnf.w"], "transformer.ln_f.bias": P["head.lnf.b"],
          "lm_head.weight": P["head.lm.w"]}
    ours_of = {}
    for l in range(cfg.layers):
        p, q = f"layers.{l}.", f"transformer.h.{l}."
        # HF Conv1D stores [in, out] = the transpose of our [out, in]
        pairs = {"ln_1.weight": "ln1.w", "ln_1.bias": "ln1.b", "attn.c_attn.weight": "attn.qkv.w",
                 "attn.c_attn.bias": "attn.qkv.b", "attn.c_proj.weight": "attn.proj.w",
                 "attn.c_proj.bias": "attn.proj.b", "ln_2.weight": "ln2.w", "ln_2.bias": "ln2.b",
                 "mlp.c_fc.weight": "mlp.fc1.w", "mlp.c_fc.bias": "mlp.fc1.b",
                 "mlp.c_proj.weight": "mlp.fc2.w", "mlp.c_proj.bias": "mlp.fc2.b"}
        for hk, ok in pairs.items():
            t = P[p + ok]
            sd[q + hk] = t.t() if hk.endswith("weight") and t.dim() == 2 else t
            ours_of[q + hk] = p + ok
    ours_of.update({"transformer.wte.weight": "embed.wte", "transformer.wpe.weight": "embed.wpe",
                    "transformer.ln_f.weight": "head.lnf.w", "transformer.ln_f.bias": "head.lnf.b",
                    "lm_head.weight": "head.lm.w"})
    missing, unexpected = model.load_state_dict({k: v.contiguous() for k, v in sd.items()}, strict=False)
    assert not unexpected and all("attn.bias" in k or "masked_bias" in k for k in missing), (missing, unexpected)
    losses = []
    for i in range(N):
        logits = model(input_ids=tok[i]).logits
        loss = F.cross_entropy(logits.reshape(-1, cfg.vocab), tgt[i].reshape(-1))
        (loss / N).backward()
        losses.append(loss.detach())
    assert rel(seq.losses, torch.stack(losses)) < 1e-13
    for hk, prm in model.named_parameters():
        g = prm.grad
        ok = ours_of[hk]
        ref = seq.grads[ok]
        if g.dim() == 2 and hk.startswith("transformer.h."):
            g = g.t()
        assert rel(ref, g) < 1e-11, hk


# --------------------------------------------------------------------------
# 3. the single update == torch.optim.AdamW
# --------------------------------------------------------------------------
@pytest.mark.parametrize("step", [1, 3])
def test_adamw_matches_torch(step):
    g = torch.Generator().manual_seed(0)
    cfg = go.OracleConfig(1, 8, 1, 4, 8, 1, lr=3e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)
    p0 = {"a": torch.randn(17, generator=g), "b": torch.randn(3, 5, generator=g)}
    grads_seq = [{k: torch.randn_like(v) for k, v in p0.items()} for _ in range(step)]
    prm = {k: v.clone().requires_grad_(True) for k, v in p0.items()}
    opt = torch.optim.AdamW(list(prm.values()), lr=cfg.lr, betas=(cfg.beta1, cfg.beta2), eps=cfg.eps,
                            weight_decay=cfg.weight_decay)
    cur = {k: v.clone() for k, v in p0.items()}
    m = {k: torch.zeros_like(v) for k, v in p0.items()}
    v_ = {k: torch.zeros_like(v) for k, v in p0.items()}
    for i, gs in enumerate(grads_seq, start=1):
        for k in prm:
            prm[k].grad = gs[k].clone()
        opt.step()
        cur, m, v_ = go.adamw_update(cur, gs, m, v_, cfg, i)
    for k in prm:
        assert rel(cur[k], prm[k].detach()) < 1e-15
