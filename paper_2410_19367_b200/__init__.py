"""B200-native BitPipe (arXiv 2410.19367).

Layers:
  * :mod:`.schedule` -- drop-in restatement of the reference ``pipesched``
    schedule generator / stage partitioner (host, pure Python);
  * :mod:`.model`    -- GPT/BERT configs, parameter layout, stage partition;
  * :mod:`.runtime`  -- the train-step executor: per-logical-device CUDA
    streams driving the C-ABI library ``libbitpipe_b200.so`` (sm_100a
    kernels, P2P slots, eager replica-pair gradient sync, fused Adam).

The reference's public schedule API is re-exported at package level.
"""
from .schedule import *  # noqa: F401,F403
from .schedule import __all__ as _sched_all

__all__ = list(_sched_all)
__version__ = "0.1.0"
