#!/usr/bin/env python3
"""TEST INFRASTRUCTURE: golden values for the C5 substitutes,
produced by the UNMODIFIED reference (oracle/_ref):

  random_regular(100, 3, 7), p=3, C4 angles: max width 27, reference-feasible
    -> energy and per-edge terms of NaiveBackend (tests/golden/wide.json);
  random_regular(100, 3, 10): max width 32 -> the reference's refusal message
    at its default cap 30 (the device runs it with cap 32; no reference value
    exists, so its tests compare complex64 against complex128).

Run: python oracle/gen_golden_wide.py   (needs oracle/_ref, ~30 s on 8 cores)
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import oracle as O  # noqa: E402

G, B = [0.30, 0.25, 0.20], [0.35, 0.30, 0.25]
out = {"angles": {"gammas": G, "betas": B}}
e7 = O.ref_random_regular(100, 3, 7)
en, _, nrec, peak = O.ref_energy(100, e7, G, B, "naive", jobs=os.cpu_count() or 1)
terms, _ = O.ref_edge_terms(100, e7, G, B, "naive", jobs=os.cpu_count() or 1)
out["seed7"] = {"n": 100, "seed": 7, "p": 3, "energy_naive": en, "n_records": nrec,
                "peak_tensor_bytes": peak,
                "terms_naive": [[float(t.real), float(t.imag)] for t in terms]}
e10 = O.ref_random_regular(100, 3, 10)
try:
    O.ref_energy(100, e10, G, B, "naive", jobs=os.cpu_count() or 1)
    out["seed10"] = {"refused": False}
except O.OracleError as ex:
    out["seed10"] = {"n": 100, "seed": 10, "p": 3, "refused": True, "message": str(ex)}
with open(os.path.join(os.path.dirname(HERE), "tests", "golden", "wide.json"), "w") as f:
    json.dump(out, f, indent=1)
print(out["seed7"]["energy_naive"], out["seed10"])
