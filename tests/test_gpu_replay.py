"""The headline measurement path and the new report/multi-GPU surfaces,
checked on the device against the reference's golden values:

* the CUDA-graph replay (qtng_plan_run_device -- bench.py's `value`) leaves
  terms bit-identical to the reference's NaiveBackend (C2, C4), read back with
  qtng_plan_terms after several replays (the per-level tile counters the last
  warp resets must survive replays);
* merged schedules (merge_buckets, engine.cpp:306-358) at C2 and C4: terms
  bit-identical to the reference's naive merged run, merges_applied/skipped
  equal to its counters (tests/golden/merged.json);
* the one-shot report (peak_tensor_bytes, records) equals the reference's;
* qtng_energy_multi on one device (the NCCL reduce path with a
  single-rank communicator) == the 1-GPU energy.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _terms(rec, key="terms_naive"):
    return np.array([complex(x, y) for x, y in rec[key]])


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_graph_replay_terms_bit_exact(q, ctx, golden, name):
    c = golden["configs"][name]
    g = q.random_regular(c["n"], 3, c["seed"])
    a = q.Angles(c["gammas"], c["betas"])
    plan = q.Plan(g, len(c["gammas"]), ctx=ctx)
    first = plan.execute(a)  # uploads the gate table
    assert np.array_equal(first, _terms(c))
    for n_runs in (1, 3, 5):
        assert plan.run_device(n_runs) > 0
        t = plan.terms()
        assert np.array_equal(t, _terms(c)), n_runs
    e = 0.5 * g.m
    for x in plan.terms().real:
        e -= 0.5 * x
    assert abs(e - c["energy_naive"]) <= 1e-12 * c["energy_naive"]


def test_graph_replay_after_new_angles(q, ctx, golden):
    c = golden["configs"]["C2"]
    g = q.random_regular(c["n"], 3, c["seed"])
    plan = q.Plan(g, 4, ctx=ctx)
    other = q.Angles([0.1, 0.2, 0.3, 0.4], [0.5, 0.4, 0.3, 0.2])
    t_other = plan.execute(other)
    plan.run_device(2)
    assert np.array_equal(plan.terms(), t_other)
    plan.execute(q.Angles(c["gammas"], c["betas"]))
    plan.run_device(2)
    assert np.array_equal(plan.terms(), _terms(c))


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_merged_energy_matches_reference(q, ctx, golden_merged, name):
    c = golden_merged[name]
    g = q.random_regular(c["n"], 3, c["seed"])
    res = q.energy_expectation(g, q.Angles(c["gammas"], c["betas"]), q.GpuBackend(ctx),
                               merged=True)
    ref = _terms(c)
    assert np.max(np.abs(res.terms - ref)) <= 1e-12
    assert abs(res.energy - c["energy_naive"]) <= 1e-10 * c["energy_naive"]
    # the multi-sum level kernel keeps the naive loop's ascending order
    assert np.array_equal(res.terms, ref)
    assert res.energy == c["energy_naive"]
    assert res.report.merges_applied == sum(c["merges_applied"])
    assert res.report.merges_skipped == sum(c["merges_skipped"])


def test_merged_plan_replay(q, ctx, golden_merged):
    c = golden_merged["C2"]
    g = q.random_regular(c["n"], 3, c["seed"])
    plan = q.Plan(g, 4, merged=True, ctx=ctx)
    assert np.array_equal(plan.execute(q.Angles(c["gammas"], c["betas"])), _terms(c))
    plan.run_device(3)
    assert np.array_equal(plan.terms(), _terms(c))


def test_energy_report_matches_reference(q, ctx, golden):
    c = golden["configs"]["C2"]
    g = q.random_regular(c["n"], 3, c["seed"])
    res = q.energy_expectation(g, q.Angles(c["gammas"], c["betas"]), q.GpuBackend(ctx),
                               records=True)
    assert res.energy == c["energy_naive"]
    rep = res.report
    assert rep.peak_tensor_bytes == c["peak_tensor_bytes"]
    assert len(rep.records) == c["n_records"]
    assert (rep.merges_applied, rep.merges_skipped) == (0, 0)
    widths = {}
    for r in rep.records:
        widths.setdefault((r.edge_u, r.edge_v), []).append(r.width)
        assert r.ops == 1 << r.width and r.elapsed_s > 0
    for i, (u, v) in enumerate(g.edges.tolist()):
        assert widths[(u, v)] == c["simulated_widths"][i]


def test_partial_selection_has_no_energy(q, ctx, golden):
    c = golden["configs"]["C1"]
    g = q.random_regular(c["n"], 3, c["seed"])
    a = q.Angles(c["gammas"], c["betas"])
    res = q.energy_expectation(g, a, q.GpuBackend(ctx), edges=[3, 1])
    assert math.isnan(res.energy)
    assert np.array_equal(res.terms, _terms(c)[[3, 1]])
    full = q.energy_expectation(g, a, q.GpuBackend(ctx), edges=list(range(g.m)))
    assert full.energy == c["energy_naive"]


def test_energy_multi_single_device(q, ctx, golden):
    c = golden["configs"]["C2"]
    g = q.random_regular(c["n"], 3, c["seed"])
    a = q.Angles(c["gammas"], c["betas"])
    res, ms = q.energy_multi(g, a, [ctx])
    assert res.energy == c["energy_naive"]
    assert np.array_equal(res.terms, _terms(c))
    assert ms.shape == (1,) and ms[0] > 0
    # refusals surface exactly like energy_expectation's
    with pytest.raises(q.ScheduleError) as ei:
        q.energy_multi(g, a, [ctx], cfg=q.EngineConfig(20))
    with pytest.raises(q.ScheduleError) as ej:
        q.energy_expectation(g, a, q.GpuBackend(ctx), cfg=q.EngineConfig(20))
    assert str(ei.value) == str(ej.value)


def test_precision_is_per_call(q, ctx, golden):
    """c64 and c128 plans interleave on one context (no context-global mode)."""
    c = golden["configs"]["C2"]
    g = q.random_regular(c["n"], 3, c["seed"])
    a = q.Angles(c["gammas"], c["betas"])
    p64 = q.Plan(g, 4, cfg=q.EngineConfig(dtype="c64"), ctx=ctx)
    p128 = q.Plan(g, 4, ctx=ctx)
    t64 = p64.execute(a)
    assert np.array_equal(p128.execute(a), _terms(c))
    assert np.max(np.abs(t64 - _terms(c))) <= 1e-5
    r64 = q.energy_expectation(g, a, q.GpuBackend(ctx), cfg=q.EngineConfig(dtype="c64"))
    assert abs(r64.energy - c["energy_naive"]) <= 1e-5 * c["energy_naive"]
    assert q.energy_expectation(g, a, q.GpuBackend(ctx)).energy == c["energy_naive"]


def test_plan_outlives_its_context(q, golden):
    """A plan keeps its context alive (garbage-collected bindings may destroy
    the context first): it still executes, and freeing it frees the context."""
    c = golden["configs"]["C1"]
    g = q.random_regular(c["n"], 3, c["seed"])
    own = q.Context(0)
    plan = q.Plan(g, 1, ctx=own)
    own.close()
    t = plan.execute(q.Angles(c["gammas"], c["betas"]))
    assert np.array_equal(t, _terms(c))
    plan.close()
