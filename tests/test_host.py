"""Host planner (CPU): the schedule the device executes must be the reference's
schedule -- same graph, elimination order, bucket membership/member order,
routing (simulated widths) -- pinned by fingerprints and golden lists from
the unmodified reference.  Mirrors proj/tests/test_graph.cpp,
test_ordering.cpp, test_network.cpp and the schedule parts of test_engine.cpp."""
import numpy as np
import pytest

import oracle as O


def fingerprints(q, g, a):
    order, init, widths = [], [], []
    for i in range(g.m):
        s = q.edge_schedule(g, i, a)
        for b in s.buckets:
            order += b.sum_vars
            init += b.sum_vars + [-2]
            for t in b.tensors:
                init += t.vars + [-3]
            init += [-4]
        order.append(-1)
        widths += q.simulate_widths(g, i, a.depth()) + [-5]
    return {"graph_edges": "%016x" % O.fnv1a_int64(g.edges.reshape(-1)),
            "elim_orders": "%016x" % O.fnv1a_int64(order),
            "initial_buckets": "%016x" % O.fnv1a_int64(init),
            "simulated_widths": "%016x" % O.fnv1a_int64(widths)}


@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_schedule_fingerprints(q, golden, name):
    c = golden["configs"][name]
    g = q.random_regular(c["n"], 3, c["seed"])
    assert g.edges.tolist() == c["edges"]
    fp = fingerprints(q, g, q.Angles(c["gammas"], c["betas"]))
    for k, v in fp.items():
        assert v == c["fingerprints"][k], k


def test_acceptance_graphs_and_schedules(q, golden):
    for rec in golden["acceptance"]:
        g = q.random_regular(rec["n"], 3, rec["seed"])
        assert g.edges.tolist() == rec["edges"]
        fp = fingerprints(q, g, q.Angles(rec["gammas"], rec["betas"]))
        assert fp["elim_orders"] == rec["fingerprints"]["elim_orders"]
        assert fp["simulated_widths"] == rec["fingerprints"]["simulated_widths"]


def test_c1_schedule_structure(q, golden, golden_schedule_c1):
    c = golden["configs"]["C1"]
    g = q.random_regular(c["n"], 3, c["seed"])
    a = q.Angles(c["gammas"], c["betas"])
    for i, ref in enumerate(golden_schedule_c1):
        s = q.edge_schedule(g, i, a)
        assert [[b.sum_vars, [t.vars for t in b.tensors]] for b in s.buckets] == \
            [[b["sum_vars"], b["tensors"]] for b in ref["buckets"]]
        assert list(g.edges[i]) == ref["edge"]


def test_c2_widths_and_counts(q, golden):
    c = golden["configs"]["C2"]
    g = q.random_regular(c["n"], 3, c["seed"])
    widths = [q.simulate_widths(g, i, 4) for i in range(g.m)]
    assert widths == c["simulated_widths"]
    assert sum(len(w) for w in widths) == c["n_records"] == 7857
    assert max(max(w) for w in widths) == c["max_width"] == 26


def test_gate_values_match_reference(q, golden):
    """Initial tensor data of every bucket equals the reference's gate_matrix
    values (circuit.cpp:38-74) bit for bit."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    c = golden["configs"]["C1"]
    g = q.random_regular(c["n"], 3, c["seed"])
    a = q.Angles(c["gammas"], c["betas"])
    for i in range(g.m):
        ints, data, nb = O.ref_edge_schedule(c["n"], g.edges, c["gammas"], c["betas"], i)
        mi, mn, md = q.edge_schedule(g, i, a).flatten()
        assert np.array_equal(mi[:mn], ints) and np.array_equal(md, data)


def test_edge_costs_are_algorithmic_bytes(q, golden):
    c = golden["configs"]["C2"]
    g = q.random_regular(c["n"], 3, c["seed"])
    costs = q.edge_costs(g, 4)
    assert costs.shape == (45,)
    assert abs(costs.sum() - 1.9769458064e10) < 1.0  # 1.977e10 B
    assert costs.max() / costs.sum() == pytest.approx(0.129, abs=0.002)


def test_refusals_host_preflight(q, golden):
    for ref in golden["refusals"]:
        g = q.random_regular(ref["n"], 3, ref["seed"])
        with pytest.raises(q.ScheduleError) as ei:
            q.validate_energy(g, len(ref["gammas"]), cfg=q.EngineConfig(ref["max_width"]))
        assert str(ei.value) == ref["message"]
    c = golden["configs"]["C2"]
    q.validate_energy(q.random_regular(30, 3, c["seed"]), 4, cfg=q.EngineConfig(27))


def test_graph_errors(q):
    with pytest.raises(q.InvalidInputError, match="degree must be smaller"):
        q.random_regular(3, 3, 1)
    with pytest.raises(q.InvalidInputError, match="must be even"):
        q.random_regular(5, 3, 1)
    with pytest.raises(q.InvalidInputError, match="self-loop"):
        q.make_graph(3, [(1, 1)])
    with pytest.raises(q.InvalidInputError, match="duplicate"):
        q.make_graph(3, [(0, 1), (1, 0)])
    with pytest.raises(q.InvalidInputError, match="out of range"):
        q.make_graph(3, [(0, 3)])
    g = q.make_graph(4, [(2, 1), (0, 3)])
    assert g.edges.tolist() == [[0, 3], [1, 2]]


def test_k4_graph(q):
    # test_engine.cpp:321-333 uses random_regular(4, 3, 0) == K4
    g = q.random_regular(4, 3, 0)
    assert g.edges.tolist() == [[0, 1], [0, 2], [0, 3], [1, 2], [1, 3], [2, 3]]


def test_angles_and_config(q, monkeypatch):
    with pytest.raises(q.InvalidInputError):
        q.Angles([0.1], []).validate()
    with pytest.raises(q.InvalidInputError, match="non-finite gamma"):
        q.Angles([float("nan")], [0.1]).validate()
    monkeypatch.setenv("QTNSIM_MAX_WIDTH", "12")
    assert q.EngineConfig.from_env().max_result_width == 12
    assert q.EngineConfig().max_result_width == 30


def test_merged_schedule_keeps_widths_bounded(q):
    # test_engine.cpp:236-246: merging never grows the widest bucket
    g = q.random_regular(12, 3, 41)
    for i in range(g.m):
        wu = q.simulate_widths(g, i, 2, merged=False)
        wm = q.simulate_widths(g, i, 2, merged=True)
        assert max(wm) <= max(wu)
        assert len(wm) <= len(wu)


def test_edge_work_is_the_reference_op_count(q, golden):
    # per lightcone: sum over buckets of 2^width * max(1, members-1) + adds;
    # summed over C2 it bounds the reference's ops (sum 2^width) from above
    c = golden["configs"]["C2"]
    g = q.random_regular(c["n"], 3, c["seed"])
    w = q.edge_work(g, 4)
    assert w.shape == (g.m,) and (w > 0).all()
    ops = q.plan_stats(g, 4).sum_ops
    assert w.sum() >= ops
    assert w.argmax() == q.edge_costs(g, 4).argmax()


@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_merged_schedules_match_reference(q, golden_merged, name):
    """merge_buckets (engine.cpp:306-358): every edge's merged schedule --
    bucket order, sum vars, member order -- its simulated widths and its
    merges_applied/merges_skipped counters equal the reference's
    (tests/golden/merged.json, oracle/gen_golden_merged.py)."""
    c = golden_merged[name]
    g = q.random_regular(c["n"], 3, c["seed"])
    a = q.Angles(c["gammas"], c["betas"])
    fp_b, fp_w, applied, skipped = [], [], [], []
    for i in range(g.m):
        s = q.edge_schedule(g, i, a, merged=True)
        for b in s.buckets:
            fp_b += b.sum_vars + [-2]
            for t in b.tensors:
                fp_b += t.vars + [-3]
            fp_b += [-4]
        fp_b.append(-1)
        fp_w += q.simulate_widths(g, i, a.depth(), merged=True) + [-5]
        applied.append(s.merges_applied)
        skipped.append(s.merges_skipped)
    assert "%016x" % O.fnv1a_int64(fp_b) == c["merged_buckets"]
    assert "%016x" % O.fnv1a_int64(fp_w) == c["merged_widths"]
    assert applied == c["merges_applied"]
    assert skipped == c["merges_skipped"]


def test_merged_schedules_live_reference(q, golden):
    """Merged C1 and a handful of C2 edges against the live reference build."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    for name, sel in (("C1", None), ("C2", [0, 7, 22, 31, 44])):
        c = golden["configs"][name]
        g = q.random_regular(c["n"], 3, c["seed"])
        a = q.Angles(c["gammas"], c["betas"])
        for i in (range(g.m) if sel is None else sel):
            ints, data, nb = O.ref_edge_schedule(c["n"], g.edges, c["gammas"], c["betas"], i,
                                                 merged=True)
            s = q.edge_schedule(g, i, a, merged=True)
            mi, mn, md = s.flatten()
            assert np.array_equal(mi[:mn], ints) and np.array_equal(md, data), (name, i)
            assert (s.merges_applied, s.merges_skipped) == O.ref_merge_counts(
                c["n"], g.edges, c["gammas"], c["betas"], i)


def test_lpt_shards_on_predicted_work(q, golden):
    """qtng_shard_edges: LPT placement of the lightcones by predicted work --
    every edge placed once, loads within LPT's bound, deterministic."""
    c = golden["configs"]["C2"]
    g = q.random_regular(c["n"], 3, c["seed"])
    w = q.edge_work(g, 4)
    for k in (1, 2, 4, 8):
        own = q.shard_edges(g, 4, k)
        assert own.shape == (g.m,) and own.min() >= 0 and own.max() < k
        loads = np.array([w[own == r].sum() for r in range(k)])
        # LPT: max load <= mean + the largest single job
        assert loads.max() <= loads.mean() + w.max() + 1e-6
        assert np.array_equal(own, q.shard_edges(g, 4, k))
    assert (q.shard_edges(g, 4, 1) == 0).all()


def _sched(q, buckets):
    return q.ContractionSchedule([q.Bucket(s, [q.Tensor(f"t{i}_{k}", v, np.asarray(d, complex))
                                               for k, (v, d) in enumerate(ts)])
                                  for i, (s, ts) in enumerate(buckets)])


def test_merge_nested_var_sets_collapse(q):
    # test_engine.cpp:173-195
    r = 1.0 / np.sqrt(2.0)
    s = _sched(q, [([0], [([0, 1], [r, 0, 0, r])]), ([1], [([1, 2], [1, 0, 0, 1])]),
                   ([2], [([2], [1, 1])])])
    m = q.merge_buckets(s)
    assert len(m.buckets) < len(s.buckets) and m.merges_applied >= 1


def test_merge_blocked_by_non_nested_kept_vars(q):
    # test_engine.cpp:197-218: bucket 0 keeps {3,4}; no single later bucket covers both
    s = _sched(q, [([0], [([0, 3, 4], [1] * 8)]), ([3], [([3], [3, 4])]), ([4], [([4], [1, 2])])])
    m = q.merge_buckets(s)
    assert len(m.buckets[0].tensors) == 1 and m.buckets[0].tensors[0].label == "t0_0"
    assert m.buckets[0].sum_vars == [0]


def test_merge_unrelated_buckets_not_chained(q):
    # test_engine.cpp:220-234
    s = _sched(q, [([0], [([0], [1, 2])]), ([1], [([1], [3, 4])])])
    m = q.merge_buckets(s)
    assert len(m.buckets) == 2 and m.merges_applied == 0


def test_merge_explicit_equals_edge_schedule_merge(q):
    """merge_buckets on an unmerged edge schedule == edge_schedule(merged=True)."""
    g = q.random_regular(10, 3, 13)
    a = q.Angles([0.6, 0.2], [0.1, 0.5])
    for i in range(g.m):
        m = q.merge_buckets(q.edge_schedule(g, i, a))
        e = q.edge_schedule(g, i, a, merged=True)
        assert [(b.sum_vars, [t.vars for t in b.tensors]) for b in m.buckets] == \
            [(b.sum_vars, [t.vars for t in b.tensors]) for b in e.buckets]
        assert (m.merges_applied, m.merges_skipped) == (e.merges_applied, e.merges_skipped)
        # test_engine.cpp:265-273: merged buckets are at least as wide as their sums
        for b in m.buckets:
            if len(b.sum_vars) > 1:
                assert len({v for t in b.tensors for v in t.vars}) >= len(b.sum_vars)
