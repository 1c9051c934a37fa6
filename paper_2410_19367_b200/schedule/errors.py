"""Exception taxonomy of the schedule layer and the train-step runtime.

The class names and the inheritance tree are part of the drop-in contract:
code written against the reference ``pipesched`` package catches these by
name (reference: ``pkg/src/pipesched/errors.py:4-91``).  Every class below
has the same parent as its reference counterpart.
"""
from __future__ import annotations

__all__ = [
    "PipeschedError", "ConfigError", "InvalidTopology", "NonPositiveBandwidth",
    "ScheduleError", "InsufficientMicroBatches", "InvalidChunking",
    "OddChunkCount", "OddDeviceCount", "MergeConflict", "SimulationError",
    "UnmappedDevice", "DeadlockDetected", "EmptyTimeline",
    "UnsupportedCombination", "EmptySpace", "RuntimeVerificationError",
    "ShapeMismatch", "ProtocolViolation",
]


class PipeschedError(Exception):
    """Root of every domain error raised by this framework."""


# configuration ---------------------------------------------------------------
class ConfigError(PipeschedError):
    """A configuration value is malformed or contradicts another one."""


class InvalidTopology(ConfigError):
    """P != W*D, or the node size does not divide the device count."""


class NonPositiveBandwidth(ConfigError):
    """Some bandwidth is <= 0."""


# schedule construction -------------------------------------------------------
class ScheduleError(PipeschedError):
    """A schedule could not be constructed or failed validation."""


class InsufficientMicroBatches(ScheduleError):
    """Too few micro-batches for the warm-up ramp (1F1B family needs N >= D)."""


class InvalidChunking(ScheduleError):
    """N does not decompose into the chunking the approach requires."""


class OddChunkCount(ScheduleError):
    """The V shape pairs descending and ascending legs: v must be even."""


class OddDeviceCount(ScheduleError):
    """Two opposite pipelines only interlock on an even number of devices."""


class MergeConflict(ScheduleError):
    """A device/time cell was claimed twice by a slot-grid union."""


# execution / simulation ------------------------------------------------------
class SimulationError(PipeschedError):
    """An execution model could not make progress or was misused."""


class UnmappedDevice(SimulationError):
    """A logical device has no physical placement."""


class DeadlockDetected(SimulationError):
    """Dataflow plus per-device order contains a cycle.

    ``cycle`` carries the tasks found blocked (device heads or the lowest
    priority stuck tasks), so callers can print a diagnosis.
    """

    def __init__(self, message: str, cycle=None):
        super().__init__(message)
        self.cycle = [] if not cycle else list(cycle)


class EmptyTimeline(SimulationError):
    """A timeline query was made on a run with no events."""


# analysis --------------------------------------------------------------------
class UnsupportedCombination(PipeschedError):
    """No closed form exists for this approach / parameter combination."""


class EmptySpace(PipeschedError):
    """A search was asked to choose from an empty configuration space."""


# numeric runtime -------------------------------------------------------------
class RuntimeVerificationError(PipeschedError):
    """Base class for train-step protocol and shape errors."""


class ShapeMismatch(RuntimeVerificationError):
    """Tensor shapes disagree with the model / stage partition."""


class ProtocolViolation(RuntimeVerificationError):
    """A task ran before its input arrived, or a message had no consumer."""
