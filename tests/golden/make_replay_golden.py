"""Generates tests/golden/replay_*.json.gz: the reference's own scenario
loader and replay (oracle/_ref/libkvtier_ref.so, ref_replay_dump in
oracle/ref_capi.cpp) run on its shipped scenarios, written as the expanded
scenario (tiers, params, space, profiles, truth curves, order, trace) plus
the replay's records, actions, final placements and metrics. Run here (the
container with /root/reference); the fixtures travel with the repo.

  python tests/golden/make_replay_golden.py
"""
import ctypes as C
import gzip
import json
import os
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "..", "..", "oracle", "_ref", "libkvtier_ref.so")
SCEN = "/root/reference/proj/scenarios"

# (fixture name, scenario, loader overrides)
CASES = [
    ("fig2_warm", "fig2", []),
    ("fig2_cold", "fig2", ["warm_start=false"]),
    ("bimodal_warm", "bimodal", []),
    ("bimodal_cold", "bimodal", ["warm_start=false"]),
    ("drift_truth_cold", "drift", ["drift.enabled=false", "warm_start=false"]),
    ("drift_warm", "drift", []),
    ("drift_cold", "drift", ["warm_start=false"]),
    ("drift_window", "drift", ["drift.window_size=8", "drift.threshold=0.2"]),
    ("drift_noise", "drift", ["drift.noise=0.05"]),
    ("bimodal_msb", "bimodal", ["warm_start=false", "miss_store_bottom=true"]),
    ("bimodal_qargmax", "bimodal", ["warm_start=false", "policy=joint-qargmax"]),
    ("bimodal_lru", "bimodal", ["warm_start=false", "policy=lru"]),
    ("bimodal_fixed", "bimodal", ["policy=fixed:keydiff:0.4"]),
    ("bimodal_impress", "bimodal", ["warm_start=false", "policy=impress:0.3"]),
    ("fig2_prefill", "fig2", ["policy=prefill"]),
    ("drift_lru", "drift", ["policy=lru"]),
]


def main():
    lib = C.CDLL(LIB)
    lib.ref_replay_dump.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_char_p), C.c_int32]
    lib.ref_last_error.restype = C.c_char_p
    for name, scen, ov in CASES:
        arr = (C.c_char_p * max(1, len(ov)))(*[o.encode() for o in ov])
        with tempfile.TemporaryDirectory() as d:
            out = os.path.join(d, "r.json")
            rc = lib.ref_replay_dump(os.path.join(SCEN, scen + ".json").encode(), out.encode(), arr, len(ov))
            if rc != 0:
                raise RuntimeError(f"{name}: {lib.ref_last_error().decode()}")
            doc = json.load(open(out))
        doc["case"] = {"name": name, "scenario": scen + ".json", "overrides": ov}
        path = os.path.join(HERE, f"replay_{name}.json.gz")
        with gzip.open(path, "wt") as f:
            json.dump(doc, f)
        r = doc["result"]
        print(name, len(doc["trace"]), "requests", len(r.get("actions", [])), "actions", "miss",
              r["metrics"]["miss_fraction"], os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
