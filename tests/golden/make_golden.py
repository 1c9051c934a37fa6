"""Generate the schedule golden fixtures FROM THE REFERENCE (run in the build
container, where /root/reference exists; the GPU box only reads the output).

Outputs (committed):
  * ``schedule_hashes.json`` -- sha256(dump_schedule(...)) of the reference
    builders over a broad sweep (approach x D x N x v x early_forward x
    layout policy), or the exception class name the reference raises;
  * ``schedules.json.gz``    -- full reference dumps for the configs the GPU
    parity tests execute (they cannot import the reference on the box).

Usage:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    import pipesched  # noqa: F401
    from pipesched import builders, fusion, schedules
    return pipesched, builders, fusion, schedules


def sweep_specs():
    """(label, kwargs) pairs.  kwargs are interpreted by ``run_ref`` / the
    tests' ``run_ours`` identically."""
    out = []
    for D in (2, 4, 6, 8, 12, 16):
        for N in sorted({D, 2 * D, 3 * D, 4 * D, D + 2, 2 * D + 1}):
            for v in (2, 4):
                out.append({"approach": "bitpipe", "D": D, "N": N, "v": v})
                if N >= 2 * D:
                    out.append({"approach": "bitpipe-early-forward", "D": D, "N": N, "v": v})
            out.append({"approach": "chimera", "D": D, "N": N})
            out.append({"approach": "dapple-1f1b", "D": D, "N": N})
            out.append({"approach": "gpipe", "D": D, "N": N})
            out.append({"approach": "interleaved-looping", "D": D, "N": N, "v": 2})
            out.append({"approach": "v-shaped", "D": D, "N": N, "v": 2})
    for D, g in ((2, 0), (4, 3), (8, 10), (12, 19)):
        for N in (D, 2 * D, 3 * D, 4 * D):
            out.append({"approach": "bitpipe", "D": D, "N": N, "v": 2,
                        "policy": ["unit-1f1b", False, g]})
    for D in (2, 4, 8):
        for N in (D, 2 * D):
            for pol in (["backward-first", True, 0], ["unit-1f1b", False, 0],
                        ["unit-1f1b", True, 1]):
                out.append({"approach": "bitpipe", "D": D, "N": N, "v": 2, "policy": pol})
    for D in (2, 4, 8):
        for n in (1, 3, 5):
            out.append({"approach": "merge-v-shaped", "D": D, "N": n})
    return out


def label(spec: dict) -> str:
    """Stable text key, e.g. ``D=4;N=8;approach=bitpipe;policy=unit-1f1b:0:3;v=2``."""
    def fmt(k, x):
        return ":".join(str(int(e)) if isinstance(e, bool) else str(e) for e in x) if k == "policy" else str(x)
    return ";".join(f"{k}={fmt(k, spec[k])}" for k in sorted(spec))


def parse_label(text: str) -> dict:
    spec = {}
    for kv in text.split(";"):
        k, x = kv.split("=", 1)
        if k == "policy":
            pri, defer, g = x.split(":")
            spec[k] = [pri, bool(int(defer)), int(g)]
        elif k == "approach":
            spec[k] = x
        else:
            spec[k] = int(x)
    return spec


def run_ref(spec: dict):
    ps, B, F, S = _ref()
    D, N = spec["D"], spec["N"]
    a = spec["approach"]
    if a == "merge-v-shaped":
        dn = ps.build_v_shaped(D, N, 2, S.Direction.DOWN)
        up = ps.build_v_shaped(D, N, 2, S.Direction.UP)
        return ps.merge_bidirectional(dn, up)
    if "policy" in spec:
        pri, defer, g = spec["policy"]
        v = spec["v"]
        maps = {d: S.v_shaped_map(D, v, d) for d in (S.Direction.DOWN, S.Direction.UP)}
        mbs = {d: B._fusion_ids(N // 2, d) for d in (S.Direction.DOWN, S.Direction.UP)}
        lay = F.fused_layout(D, v, maps, mbs, unit_size=max(1, D // 2),
                             policy=F.LayoutPolicy(pri, defer, g))
        sch = S.Schedule(ps.ApproachId.BITPIPE, D, N, v, -(-N // D), lay.per_device,
                         (maps[S.Direction.DOWN], maps[S.Direction.UP]), starts=dict(lay.starts))
        return S.validate_schedule(sch)
    approach = ps.ApproachId(a)
    return ps.build(approach, D, N, spec.get("v"), a == "bitpipe-early-forward")


def outcome(fn) -> str:
    ps, B, F, S = _ref()
    try:
        text = S.dump_schedule(fn())
    except Exception as e:  # reference error class is part of the contract
        return "error:" + type(e).__name__
    return "sha256:" + hashlib.sha256(text.encode()).hexdigest()


# configs whose full reference dump travels to the GPU box
FULL = [
    {"approach": "bitpipe", "D": 2, "N": 2, "v": 2},
    {"approach": "bitpipe", "D": 2, "N": 4, "v": 2},
    {"approach": "bitpipe", "D": 4, "N": 4, "v": 2},
    {"approach": "bitpipe", "D": 4, "N": 8, "v": 2},
    {"approach": "bitpipe", "D": 8, "N": 16, "v": 2},
    {"approach": "bitpipe", "D": 4, "N": 8, "v": 2, "policy": ["unit-1f1b", False, 3]},
    {"approach": "bitpipe", "D": 8, "N": 16, "v": 2, "policy": ["unit-1f1b", False, 10]},
    {"approach": "bitpipe", "D": 2, "N": 4, "v": 4},
    {"approach": "bitpipe-early-forward", "D": 4, "N": 8, "v": 2},
    {"approach": "chimera", "D": 4, "N": 4},
    {"approach": "dapple-1f1b", "D": 4, "N": 4},
    {"approach": "gpipe", "D": 2, "N": 4},
    {"approach": "interleaved-looping", "D": 4, "N": 4, "v": 2},
    {"approach": "interleaved-looping", "D": 2, "N": 4, "v": 2},
]


def main():
    ps, B, F, S = _ref()
    hashes = {label(s): outcome(lambda s=s: run_ref(s)) for s in sweep_specs()}
    with open(os.path.join(HERE, "schedule_hashes.json"), "w") as f:
        json.dump(hashes, f, indent=0, sort_keys=True)
    full = {label(s): S.dump_schedule(run_ref(s)) for s in FULL}
    with gzip.open(os.path.join(HERE, "schedules.json.gz"), "wt") as f:
        json.dump(full, f, sort_keys=True)
    print(f"{len(hashes)} hashes, {len(full)} full dumps")


if __name__ == "__main__":
    main()
