"""The drop-in boundary: the package re-exports the reference's public names
(``pipesched/__init__.py:23-44``) with the same signatures, plus the SPEC's
train-step entry (``run_schedule_numeric``)."""
import inspect

import pytest

import paper_2410_19367_b200 as ours

REF_ALL = ["ApproachId", "ClusterSpec", "CostModel", "ModelProfile", "message_size", "validate_cluster",
           "Direction", "Schedule", "StageMap", "Task", "TaskKind", "validate_schedule", "build", "build_1f1b",
           "build_bitpipe", "build_chimera", "build_gpipe", "build_interleaved_looping", "build_v_shaped",
           "merge_bidirectional"]


def test_reference_names_exported():
    for n in REF_ALL:
        assert n in ours.__all__ and hasattr(ours, n), n


def _params(obj):
    try:
        sig = inspect.signature(obj)
    except (TypeError, ValueError):
        return None
    return [(p.name, p.kind, p.default) for p in sig.parameters.values()]


@pytest.mark.reference
def test_surface_matches_imported_reference(ref_pipesched):
    """Every one of the reference's 20 names: same kind of object, same
    call signature (our builders add only a trailing optional ``policy``),
    same enum members, same dataclass fields."""
    import dataclasses
    import enum
    assert sorted(ref_pipesched.__all__) == sorted(REF_ALL)
    for n in ref_pipesched.__all__:
        r, o = getattr(ref_pipesched, n), getattr(ours, n)
        assert isinstance(r, type) == isinstance(o, type), n
        if isinstance(r, type) and issubclass(r, enum.Enum):
            assert [(m.name, m.value) for m in r] == [(m.name, m.value) for m in o], n
            continue
        if dataclasses.is_dataclass(r):
            assert [f.name for f in dataclasses.fields(r)] == [f.name for f in dataclasses.fields(o)], n
        rp, op = _params(r), _params(o)
        if rp is None:
            continue
        extra = [p for p in op if p not in rp]
        assert op[:len(rp)] == rp, (n, rp, op)
        assert all(p[0] == "policy" and p[2] is None for p in extra), (n, extra)  # trailing, optional


def test_train_step_entry_exported():
    from paper_2410_19367_b200.runtime import api
    sig = inspect.signature(api.train_step)
    assert list(sig.parameters)[:4] == ["schedule", "model", "batch", "seed"]
    assert api.run_schedule_numeric is api.train_step
    assert {f for f in api.StepResult.__dataclass_fields__} >= {"losses", "loss", "grads", "params"}
