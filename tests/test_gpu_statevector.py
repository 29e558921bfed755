"""Device state-vector oracle (sv.cu) vs the reference's StateVector
(proj/src/statevector.cpp) and, at the C2 headline size (30 qubits, beyond the
reference's default cap of 24), vs the tensor-network energy itself -- two
independent methods on the same device."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def test_acceptance_instances_vs_reference_statevector(q, ctx, golden):
    n_checked = 0
    for rec in golden["acceptance"]:
        if rec.get("energy_statevector") is None:
            continue
        g = q.random_regular(rec["n"], 3, rec["seed"])
        e, zz = q.statevector_energy(g, q.Angles(rec["gammas"], rec["betas"]), ctx=ctx)
        assert abs(e - rec["energy_statevector"]) <= 1e-12 * max(1.0, abs(e)), rec["name"]
        # the per-edge terms equal the tensor network's Re e_jk
        terms = np.array([x for x, _ in rec["terms_naive"]])
        assert np.max(np.abs(zz - terms)) <= 1e-12, rec["name"]
        n_checked += 1
    assert n_checked >= 10


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_live_reference_statevector(q, ctx):
    for n, seed, p in [(10, 3, 2), (14, 11, 3), (18, 2, 2)]:
        g = q.random_regular(n, 3, seed)
        gam, bet = [0.4, -0.3, 0.2][:p], [0.7, 0.1, -0.5][:p]
        ref = O.ref_statevector_energy(n, g.flat().reshape(-1, 2), gam, bet)
        e, _ = q.statevector_energy(g, q.Angles(gam, bet), ctx=ctx)
        assert abs(e - ref) <= 1e-12 * max(1.0, abs(ref)), (n, seed)


def test_zero_angles_and_cap(q, ctx):
    g = q.random_regular(12, 3, 4)
    e, zz = q.statevector_energy(g, q.Angles([0.0], [0.0]), ctx=ctx)
    assert e == pytest.approx(g.m / 2, abs=1e-13) and np.allclose(zz, 0.0, atol=1e-13)
    big = q.random_regular(30, 3, 104478)
    with pytest.raises(q.ResourceError) as ei:
        q.statevector_energy(big, q.Angles([0.1], [0.2]), ctx=ctx)
    assert str(ei.value) == "state vector of 30 qubits exceeds cap 24"


def test_c2_headline_two_methods(q, ctx, golden):
    # 30 qubits = 16 GiB of amplitudes: the C2 energy by brute force, against
    # the bucket-elimination value (bit-identical to the reference's naive)
    c = golden["configs"]["C2"]
    g = q.random_regular(c["n"], 3, c["seed"])
    e, zz = q.statevector_energy(g, q.Angles(c["gammas"], c["betas"]), cap=30, ctx=ctx)
    assert abs(e - c["energy_naive"]) <= 1e-10 * abs(c["energy_naive"])
    terms = np.array([x for x, _ in c["terms_naive"]])
    assert np.max(np.abs(zz - terms)) <= 1e-10


@pytest.mark.parametrize("seed", range(6))
def test_random_instances_two_methods(q, ctx, seed):
    # random graphs and angles: the bucket-elimination energy (fused chains,
    # pipelined one-shot path) against the device state vector
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([6, 8, 10, 12, 14, 16]))
    p = int(rng.integers(1, 4))
    g = q.random_regular(n, 3, int(rng.integers(0, 1 << 30)))
    a = q.Angles(list(rng.uniform(-np.pi, np.pi, p)), list(rng.uniform(-np.pi, np.pi, p)))
    res = q.energy_expectation(g, a, q.GpuBackend(ctx))
    e_sv, zz = q.statevector_energy(g, a, ctx=ctx)
    assert abs(res.energy - e_sv) <= 1e-10 * max(1.0, abs(e_sv)), (n, p)
    assert np.max(np.abs(res.terms.real - zz)) <= 1e-10
    assert np.max(np.abs(res.terms.imag)) <= 1e-8
