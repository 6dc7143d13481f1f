"""Golden fixtures for the staging slot region and the recovery consensus,
made by running the REFERENCE package's engine (reference engine.py).

Run in the build container (where /root/reference exists):

    python tests/golden/make_engine_golden.py

Writes tests/golden/engine_golden.json: a scripted sequence of SlotRegion
calls with each call's outcome (slot info or exception class) and the final
region file bytes; the staging blob of the golden checkpoint
(checkpoint_golden.npz, iteration 110) staged into a fresh region (sha256 of
the file); and two recovery scenarios (decision, pruned slots, trace).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = os.environ.get("BITSNAP_REF_SRC", "/root/reference/pkg/src")

# (op, args...) with payloads as hex strings
SCRIPT = [
    ["stage", 0, b"alpha-payload".hex(), 1],
    ["stage", 1, "", 1],
    ["stage", 0, bytes(range(48)).hex(), 2],
    ["stage", 0, b"late".hex(), 2],            # stale
    ["stage", 0, b"z".hex(), 3],               # backpressure: both slots VALID
    ["set_state", 0, 0, 3],                    # slot 0 PERSISTED
    ["stage", 0, b"third".hex(), 3],           # evicts the persisted slot
    ["stage", 1, (b"y" * 49).hex(), 5],        # too large
    ["stage", 1, b"beta".hex(), 4],
    ["verify", 0, 0],
    ["verify", 1, 1],
    ["clear", 1, 0],
    ["verify", 1, 0],
    ["stage", 1, b"gamma".hex(), 6],
]
REGION = {"ranks": 2, "redundancy": 2, "capacity": 48}


def _ref():
    sys.path.insert(0, REF_SRC)
    from bitsnap import engine, store, tensors
    return engine, store, tensors


def run_script(engine, path):
    region = engine.SlotRegion.create(path, **REGION)
    out = []
    for op, *a in SCRIPT:
        try:
            if op == "stage":
                s = region.stage(a[0], bytes.fromhex(a[1]), a[2])
                out.append(["ok", s.rank, s.index, s.state, s.iteration, s.length,
                            str(s.checksum)])
            elif op == "set_state":
                region.set_state(*a)
                out.append(["ok"])
            elif op == "clear":
                region.clear_slot(*a)
                out.append(["ok"])
            elif op == "verify":
                out.append(["ok", bool(region.verify(*a))])
        except Exception as exc:  # the reference's exception class is the result
            out.append(["raise", type(exc).__name__])
    status = engine.status_report(region)
    slots = [[s.rank, s.index, s.state, s.iteration, s.length, str(s.checksum)]
             for s in region.all_slots()]
    region.close()
    with open(path, "rb") as f:
        data = f.read()
    # the report names the file: keep only the lines after the first
    return {"results": out, "slots": slots, "status": status.split("\n")[1:],
            "file_hex": data.hex()}


def stage_golden_checkpoint(engine, store, path):
    g = np.load(os.path.join(HERE, "checkpoint_golden.npz"))
    man = store.CheckpointManifest.from_bytes(g["manifest1"].tobytes())
    blob = store.pack_blob(man, g["blob1"].tobytes())
    region = engine.SlotRegion.create(path, ranks=1, redundancy=2, capacity=len(blob) + 100)
    s = region.stage(0, blob, man.iteration)
    region.close()
    with open(path, "rb") as f:
        data = f.read()
    return {"capacity": len(blob) + 100, "blob_len": len(blob),
            "checksum": str(s.checksum), "file_sha256": hashlib.sha256(data).hexdigest()}


def recovery(engine, tmp):
    cases = {}
    # consensus: rank 0 holds 3 and 4, rank 1 holds 3 and a corrupt 4
    region = engine.SlotRegion.create(os.path.join(tmp, "r1.bssl"), ranks=2, redundancy=3,
                                      capacity=16)
    region.stage(0, b"r0-it3", 3)
    region.stage(0, b"r0-it4", 4)
    region.stage(1, b"r1-it3", 3)
    s = region.stage(1, b"r1-it4", 4)
    off = region._slot_offset(1, s.index) + engine.SLOT_HEADER.size
    region._mm[off] ^= 0xFF
    root = os.path.join(tmp, "stores1")
    d = engine.recover(engine.gather_reports(region, root), region, root)
    cases["consensus"] = {"chosen": d.chosen_iteration, "pruned": d.pruned,
                          "trace": d.trace,
                          "slots": [[x.rank, x.index, x.state, x.iteration]
                                    for x in region.all_slots()]}
    region.close()
    # cold start: no common iteration
    region = engine.SlotRegion.create(os.path.join(tmp, "r2.bssl"), ranks=2, redundancy=2,
                                      capacity=16)
    region.stage(0, b"a", 5)
    region.stage(1, b"b", 6)
    root = os.path.join(tmp, "stores2")
    try:
        engine.recover(engine.gather_reports(region, root), region, root)
        cases["cold"] = {"raised": None}
    except engine.ColdStartError as exc:
        cases["cold"] = {"raised": type(exc).__name__, "message": str(exc)}
    region.close()
    return cases


def main():
    engine, store, _ = _ref()
    with tempfile.TemporaryDirectory() as tmp:
        meta = {
            "generator": "tests/golden/make_engine_golden.py",
            "region": REGION,
            "script": SCRIPT,
            "script_out": run_script(engine, os.path.join(tmp, "script.bssl")),
            "checkpoint_stage": stage_golden_checkpoint(engine, store,
                                                        os.path.join(tmp, "ckpt.bssl")),
            "recovery": recovery(engine, tmp),
            "empty_checksum": str(engine.EMPTY_CHECKSUM),
        }
    with open(os.path.join(HERE, "engine_golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote engine_golden.json")


if __name__ == "__main__":
    main()
