"""The reference's own engine unit tests (proj/tests/test_engine.cpp) that
pin behaviour rather than golden numbers, run through the B200 path."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sched(q, buckets):
    return q.ContractionSchedule([q.Bucket(s, [q.Tensor(f"t{i}_{k}", v, np.asarray(d, complex))
                                               for k, (v, d) in enumerate(ts)])
                                  for i, (s, ts) in enumerate(buckets)])


def _rel(a, b):
    return abs(a - b) / max(1.0, abs(b))


@pytest.mark.parametrize("case", ["nested", "blocked", "unrelated"])
def test_merged_explicit_schedules_contract_equal(q, ctx, case):
    # test_engine.cpp:173-234: merging never changes the contracted scalar
    r = 1.0 / np.sqrt(2.0)
    s = {"nested": [([0], [([0, 1], [r, 0, 0, r])]), ([1], [([1, 2], [1, 0, 0, 1])]),
                    ([2], [([2], [1, 1])])],
         "blocked": [([0], [([0, 3, 4], [1] * 8)]), ([3], [([3], [3, 4])]), ([4], [([4], [1, 2])])],
         "unrelated": [([0], [([0], [1, 2])]), ([1], [([1], [3, 4])])]}[case]
    sched = _sched(q, s)
    be = q.GpuBackend(ctx)
    ref = q.contract_network(sched, be).scalar
    got = q.contract_network(q.merge_buckets(sched), be).scalar
    assert _rel(got, ref) < 1e-12


def test_merged_and_unmerged_qaoa_schedules_agree(q, ctx):
    # test_engine.cpp:248-263 (random angles in [0, 3), edges 0 and 5)
    rng = np.random.default_rng(31)
    be = q.GpuBackend(ctx)
    for trial in range(4):
        g = q.random_regular(8, 3, 50 + trial)
        a = q.Angles(list(rng.uniform(0, 3, 2)), list(rng.uniform(0, 3, 2)))
        for e in (0, 5):
            un = q.edge_schedule(g, e, a)
            me = q.edge_schedule(g, e, a, merged=True)
            assert len(me.buckets) <= len(un.buckets)
            ref = q.contract_network(un, be).scalar
            got = q.contract_network(me, be).scalar
            assert _rel(got, ref) < 1e-10


def test_energy_never_exceeds_maxcut_optimum_k4(q, ctx):
    # test_engine.cpp:321-333: K4's MaxCut optimum is 4
    k4 = q.random_regular(4, 3, 0)
    res = q.energy_expectation(k4, q.Angles([0.6], [0.4]), q.GpuBackend(ctx))
    assert res.energy <= 4 + 1e-10
    e_sv, _ = q.statevector_energy(k4, q.Angles([0.6], [0.4]), ctx=ctx)
    assert abs(res.energy - e_sv) < 1e-12


def test_peak_tensor_bytes_bounded_by_widest_bucket(q, ctx):
    # test_engine.cpp:422-432
    g = q.random_regular(8, 3, 23)
    rep = q.contract_network(q.edge_schedule(g, 0, q.Angles([0.9], [0.2])), q.GpuBackend(ctx))
    w = max(r.width for r in rep.records)
    assert 16 <= rep.peak_tensor_bytes <= 16 * (1 << w)


def test_small_and_degenerate_graphs(q, ctx):
    """Edge cases the reference accepts: one edge, a path, a disconnected
    graph (lightcones of separate components), and no edges at all; every
    energy equals the device state-vector oracle, and an edgeless graph has
    energy 0 (engine.cpp:549-560 with m = 0)."""
    a = q.Angles([0.7, 0.2], [0.4, 0.9])
    for n, edges in ((2, [(0, 1)]), (4, [(0, 1), (1, 2), (2, 3)]),
                     (6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)])):
        g = q.make_graph(n, edges)
        res = q.energy_expectation(g, a, q.GpuBackend(ctx))
        e_sv, _ = q.statevector_energy(g, a, ctx=ctx)
        assert abs(res.energy - e_sv) < 1e-12, (n, edges)
        plan = q.Plan(g, 2, ctx=ctx)
        assert np.array_equal(plan.execute(a), res.terms)
    g0 = q.make_graph(3, [])
    assert q.energy_expectation(g0, a, q.GpuBackend(ctx)).energy == 0.0
