"""The one-shot energy's host/device pipeline (capi.cpp energy_run): the
selected lightcones are split into chunks, each planned on the host while the
earlier chunks run, and enqueued by the context's enqueue thread.  Every
lightcone is computed by the same operations whatever the chunking, so the
energy and every term stay `==` the reference's naive values under each lane
count, ordering and split (settings are read once per process: children).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r'''
import json, sys
sys.path.insert(0, %r)
import paper_2204_06045_b200 as q
c = json.load(open(%r))["configs"][%r]
g = q.random_regular(c["n"], 3, c["seed"])
a = q.Angles(c["gammas"], c["betas"])
ctx = q.Context(0)
out = []
for _ in range(3):  # repeated calls reuse the lanes and the enqueue thread
    r = q.energy_expectation(g, a, q.GpuBackend(ctx), records=True)
    out.append({"energy": r.energy, "terms": [[float(x.real), float(x.imag)] for x in r.terms],
                "n_records": len(r.report.records)})
print(json.dumps(out))
'''


def _child(name, env):
    code = CODE % (ROOT, os.path.join(ROOT, "tests", "golden", "energies.json"), name)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
@pytest.mark.parametrize("env", [
    {"QTNG_PIPELINE": "1"},
    {"QTNG_PIPELINE": "2"},
    {"QTNG_PIPELINE": "3"},
    {"QTNG_PIPELINE": "4"},
    {"QTNG_PIPELINE": "3", "QTNG_PIPELINE_ORDER": "1"},
    {"QTNG_PIPELINE": "3", "QTNG_PIPELINE_SPLIT": "0.5,0.3,0.2"},
    {"QTNG_PIPELINE": "2", "QTNG_PIPELINE_SPLIT": "0.9,0.1"},
], ids=lambda e: ",".join(f"{k[5:]}={v}" for k, v in e.items()))
def test_pipeline_chunks_bitwise(golden, env):
    c = golden["configs"]["C2"]
    ref = [[x, y] for x, y in c["terms_naive"]]
    runs = _child("C2", env)
    for r in runs:
        assert r["terms"] == ref
        assert r["energy"] == c["energy_naive"]
        assert r["n_records"] == c["n_records"]


@pytest.mark.gpu
def test_pipeline_shared_context_threads(q, golden):
    # several host threads on ONE context: the context lock serialises the
    # device phase (the enqueue thread works for the lock holder); every call
    # returns the reference's terms
    import threading
    c = golden["configs"]["C2"]
    ref = np.array([complex(x, y) for x, y in c["terms_naive"]])
    g = q.random_regular(c["n"], 3, c["seed"])
    a = q.Angles(c["gammas"], c["betas"])
    ctx = q.Context(0)
    results, errors = [], []

    def work():
        try:
            for _ in range(3):
                results.append(q.energy_expectation(g, a, q.GpuBackend(ctx)))
        except Exception as ex:  # reported below
            errors.append(ex)

    th = [threading.Thread(target=work) for _ in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    assert len(results) == 12
    for r in results:
        assert np.array_equal(r.terms, ref)
        assert r.energy == c["energy_naive"]
