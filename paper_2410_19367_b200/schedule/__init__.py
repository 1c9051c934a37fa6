"""Schedule layer: drop-in restatement of the reference ``pipesched`` API.

``from paper_2410_19367_b200 import schedule as pipesched`` exposes the same
20 public names as ``pkg/src/pipesched/__init__.py:23-44`` with the same
signatures, values and exceptions, plus the layout engines, wire format and
analytic helpers the GPU executor and benchmarks use.
"""
from .domain import (ApproachId, BIDIRECTIONAL_APPROACHES, ClusterSpec, CostModel,
                     ModelProfile, message_size, validate_cluster)
from .plan import (Direction, Schedule, StageMap, Task, TaskKind, dump_schedule,
                   load_schedule, looping_map, schedule_from_dict, schedule_to_dict,
                   v_shaped_map, validate_schedule)
from .layout import FusedLayout, LayoutPolicy, fused_layout, list_schedule
from .builders import (PAPER_GATE_STAGE, build, build_1f1b, build_bitpipe, build_chimera,
                       build_gpipe, build_interleaved_looping, build_v_shaped,
                       merge_bidirectional, paper_policy)
from .analysis import (CommTotals, analytic_bubble_ratio, analytic_comm_count, analytic_comm_time,
                       analytic_makespan, canonical_bubble, canonical_replay, comm_accounting,
                       peak_activations, replay_times, search_bitpipe_policy)
from . import errors

__all__ = [
    # the reference's public surface (pipesched/__init__.py:23-44)
    "ApproachId", "ClusterSpec", "CostModel", "ModelProfile", "message_size",
    "validate_cluster", "Direction", "Schedule", "StageMap", "Task", "TaskKind",
    "validate_schedule", "build", "build_1f1b", "build_bitpipe", "build_chimera",
    "build_gpipe", "build_interleaved_looping", "build_v_shaped", "merge_bidirectional",
    # extensions
    "BIDIRECTIONAL_APPROACHES", "dump_schedule", "load_schedule", "schedule_to_dict",
    "schedule_from_dict", "looping_map", "v_shaped_map", "FusedLayout", "LayoutPolicy",
    "fused_layout", "list_schedule", "PAPER_GATE_STAGE", "paper_policy", "peak_activations", "search_bitpipe_policy",
    "analytic_bubble_ratio", "analytic_makespan", "canonical_bubble", "canonical_replay",
    "CommTotals", "comm_accounting", "analytic_comm_count", "analytic_comm_time", "replay_times",
    "errors",
]

__version__ = "0.1.0"
