"""CPU checks of the oracle itself (no GPU).

The reference pins no numeric values (it has no train step);
the oracle is pinned by the SPEC's schedule-independence theorem
(SPEC.md:447): executing ANY reference order with message passing must
equal the sequential baseline within 1e-9 (fp64), and by torch autograd
cross-checks of the restated model."""
import gzip
import json
import os

import pytest
import torch

from oracle.gpt_oracle import OracleConfig, run_schedule_numeric, sequential_baseline, stage_halfblocks
from paper_2410_19367_b200.model import CONFIGS, init_params, stage_partition, synthetic_batch

GOLD = os.path.join(os.path.dirname(__file__), "golden", "schedules.json.gz")


def _golden():
    with gzip.open(GOLD, "rt") as f:
        return json.load(f)


def _ocfg(cfg):
    return OracleConfig(cfg.layers, cfg.hidden, cfg.heads, cfg.seq, cfg.vocab, cfg.micro_batch, cfg.causal)


def rel(a, b):
    return ((a - b).norm() / b.norm().clamp_min(1e-300)).item()


@pytest.mark.parametrize("label", sorted(_golden()))
def test_schedule_independence(label):
    text = _golden()[label]
    cfg = CONFIGS["tiny"]
    N = json.loads(text)["N"]
    params = init_params(cfg, 3, perturb=True)
    tok, tgt = synthetic_batch(cfg, N, seed=5)
    seq = sequential_baseline(_ocfg(cfg), params, tok, tgt)
    run = run_schedule_numeric(_ocfg(cfg), text, params, tok, tgt)
    assert rel(run.losses, seq.losses) < 1e-12
    for k in params:
        assert rel(run.grads[k], seq.grads[k]) < 1e-9, k
        assert rel(run.params[k], seq.params[k]) < 1e-9, k


def test_partition_rule_matches_product():
    for cfg_name in ("tiny", "gpt-1.3b", "bert-large", "gpt-10b"):
        cfg = CONFIGS[cfg_name]
        for S in (4, 8, 16, 32):
            ours = [list(p.halfblocks) for p in stage_partition(cfg, S)]
            assert ours == stage_halfblocks(cfg.layers, S)
    # SURVEY §7 step 3 integral split examples
    assert [len(p.halfblocks) for p in stage_partition(CONFIGS["gpt-1.3b"], 16)] == [3] * 16
    assert [len(p.halfblocks) for p in stage_partition(CONFIGS["bert-large"], 8)] == [6] * 8


def test_oracle_bidirectional_mean_semantics():
    """Replica-mean of per-replica means == global mean over N."""
    cfg = CONFIGS["tiny"]
    text = _golden()["D=2;N=4;approach=bitpipe;v=2"]
    params = init_params(cfg, 1)
    tok, tgt = synthetic_batch(cfg, 4, seed=2)
    run = run_schedule_numeric(_ocfg(cfg), text, params, tok, tgt)
    # one micro-batch at a time through the sequential baseline, averaged
    acc = None
    for i in range(4):
        r = sequential_baseline(_ocfg(cfg), params, tok[i:i + 1], tgt[i:i + 1])
        acc = r.grads if acc is None else {k: acc[k] + r.grads[k] for k in acc}
    for k in acc:
        assert rel(run.grads[k], acc[k] / 4) < 1e-9
