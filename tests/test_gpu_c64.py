"""complex64 mode (north_star: "or 1e-5 for an optional complex64 mode"): the
same plans with a float2 arena and single-precision products; energies and
per-edge terms within 1e-5 of the reference's complex128 values."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

C64 = None


def _cfg(q):
    return q.EngineConfig(dtype="c64")


def _check(q, ctx, rec, tol=1e-5):
    g = q.random_regular(rec["n"], 3, rec["seed"])
    res = q.energy_expectation(g, q.Angles(rec["gammas"], rec["betas"]), q.GpuBackend(ctx),
                               cfg=_cfg(q))
    ref = rec["energy_naive"]
    assert abs(res.energy - ref) <= tol * max(1.0, abs(ref)), (rec["name"], res.energy, ref)
    terms = np.array([complex(x, y) for x, y in rec["terms_naive"]])
    assert np.max(np.abs(res.terms - terms)) <= tol
    return res


@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_configs_c64(q, ctx, golden, name):
    res = _check(q, ctx, golden["configs"][name])
    # the survey's emulated-naive complex64 values
    point = {"C1": 9.5632460415, "C2": 25.9308949239}.get(name)
    if point is not None:
        assert abs(res.energy - point) <= 1e-6 * point


def test_acceptance_c64(q, ctx, golden):
    for rec in golden["acceptance"]:
        _check(q, ctx, rec)


def test_c64_plan_and_default_restored(q, ctx, golden):
    c = golden["configs"]["C2"]
    g = q.random_regular(c["n"], 3, c["seed"])
    a = q.Angles(c["gammas"], c["betas"])
    plan = q.Plan(g, 4, cfg=_cfg(q), ctx=ctx)
    t = plan.execute(a)
    e = 0.5 * g.m - 0.5 * float(np.sum(t.real))
    assert abs(e - c["energy_naive"]) <= 1e-5 * c["energy_naive"]
    assert plan.run_device(2) > 0
    # the context precision reverts: a default energy is bit-exact again
    res = q.energy_expectation(g, a, q.GpuBackend(ctx))
    assert res.energy == c["energy_naive"]
