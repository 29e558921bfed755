"""Pinning the checkers (CPU).  The C restatement in oracle/ must reproduce the
reference's golden vectors (produced by oracle/gen_golden.py from the
unmodified reference) before it is trusted as the GPU path's oracle."""
import numpy as np
from conftest import reorder
import pytest

import oracle as O


def _tensors(b):
    return [(t["vars"], np.array(t["re"]) + 1j * np.array(t["im"])) for t in b["tensors"]]


def test_restatement_matches_reference_naive_bit_exact(golden_buckets):
    assert len(golden_buckets) >= 40
    for b in golden_buckets:
        ov, od = O.oracle_contract_bucket(_tensors(b), b["sum_vars"])
        assert ov == b["out_vars"]
        naive = np.array(b["naive_re"]) + 1j * np.array(b["naive_im"])
        assert np.array_equal(od, naive)
        matmul = reorder(np.array(b["matmul_re"]) + 1j * np.array(b["matmul_im"]), b["matmul_vars"], b["out_vars"])
        assert np.max(np.abs(od - matmul), initial=0.0) < 1e-12  # test_engine.cpp:91-104


def test_restatement_absent_sum_var():
    with pytest.raises(O.OracleError, match="absent"):
        O.oracle_contract_bucket([([0, 1], np.ones(4))], [5])


def test_statevector_restatement(golden):
    recs = [golden["configs"]["C1"]] + [r for r in golden["acceptance"] if "energy_statevector" in r]
    for r in recs:
        e = O.oracle_statevector_energy(r["n"], r["edges"], r["gammas"], r["betas"])
        assert abs(e - r["energy_statevector"]) < 1e-12
        assert abs(e - r["energy_naive"]) < 1e-8  # acceptance criterion 1


def test_restated_network_on_product_schedules(q, golden):
    """The oracle's contract_network over the product's host-built schedules
    reproduces the reference's per-edge naive terms bit for bit."""
    for rec in [golden["configs"]["C1"]] + golden["acceptance"][:6]:
        g = q.random_regular(rec["n"], 3, rec["seed"])
        a = q.Angles(rec["gammas"], rec["betas"])
        for i in range(g.m):
            sch = q.edge_schedule(g, i, a)
            ints, n, data = sch.flatten()
            s, seq, wid, peak = O.oracle_contract_network(len(sch.buckets), ints[:n], data)
            assert [s.real, s.imag] == rec["terms_naive"][i]
            assert list(wid) == q.simulate_widths(g, i, a.depth())


def test_restated_network_cap_and_liveness():
    # cap (engine.cpp:160-169)
    ints = np.array([1, 0, 1, 3, 0, 1, 2], np.int32)
    data = np.ones(16)
    with pytest.raises(O.OracleError, match="result width 2 exceeds cap 1"):
        O.oracle_contract_network(1, ints, data, max_result_width=1)
    # stray sum variable (test_engine.cpp:344-356)
    ints = np.array([1, 0, 1, 1, 0, 1, 1, 1, 2, 0, 1], np.int32)
    data = np.ones(2 * (2 + 4))
    with pytest.raises(O.OracleError, match="still live"):
        O.oracle_contract_network(2, ints, data)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_restatement_vs_live_reference():
    rng = np.random.default_rng(5)
    for trial in range(10):
        n_vars = 4 + trial % 7
        base = list(range(n_vars))
        ts = []
        for t in range(1 + trial % 4):
            vs = [v for v in base if t == 0 or rng.integers(2)] or [0]
            rng.shuffle(vs)
            ts.append((vs, rng.normal(size=1 << len(vs)) + 1j * rng.normal(size=1 << len(vs))))
        sums = sorted(rng.choice(base, size=1 + trial % 3, replace=False).tolist())
        rv, rd = O.ref_contract_bucket(ts, sums, "naive")
        ov, od = O.oracle_contract_bucket(ts, sums)
        assert rv == ov and np.array_equal(rd, od)
