"""Host-side executor logic that needs no GPU."""
import pytest
import torch

from paper_2410_19367_b200.runtime.executor import choose_deferred_stages


def test_all_stages_deferred_when_slots_fit():
    assert choose_deferred_stages({0: 10, 1: 20, 2: 30}, {0: 1, 1: 1, 2: 1}, 60) == {0, 1, 2}


def test_greedy_by_work_per_byte_under_budget():
    sizes = {0: 40, 1: 40, 2: 10, 3: 0}
    work = {0: 80, 1: 40, 2: 30, 3: 5}
    # work / byte: stage 2 (3.0), stage 0 (2.0), stage 1 (1.0); empty slot sets are never "deferred"
    assert choose_deferred_stages(sizes, work, 55) == {2, 0}
    assert choose_deferred_stages(sizes, work, 5) == set()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the CPU-only failure mode")
def test_train_step_fails_loudly_without_a_gpu():
    """No CPU fallback: the SPEC entry refuses to run without CUDA."""
    from paper_2410_19367_b200 import build_bitpipe
    from paper_2410_19367_b200.model import CONFIGS, synthetic_batch
    from paper_2410_19367_b200.runtime.api import train_step
    with pytest.raises(RuntimeError, match="CUDA"):
        train_step(build_bitpipe(2, 4), "tiny", synthetic_batch(CONFIGS["tiny"], 4))
