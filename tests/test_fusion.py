"""Fused bucket chains (device_plan.hpp "segments").

CPU: the planner's segment formation is a pure regrouping -- same buckets,
same records, same reference accounting -- with the HBM traffic of the fused
program far below the reference's per-bucket bytes, and every fused stage of
the shape the seg_kernel evaluates (main member last, one summed var).

GPU: the fused program is bit-identical to the one-op-per-bucket program and
to the reference at every segment length (QTNG_SEG_J) -- each intermediate
element is produced by the same operation sequence whether it lives in HBM
or in a register.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cfg(golden, name):
    c = golden["configs"][name]
    return c, len(c["gammas"])


@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_fusion_is_a_regrouping(q, golden, name):
    c, p = _cfg(golden, name)
    g = q.random_regular(c["n"], 3, c["seed"])
    fused, plain = q.plan_stats(g, p, fuse=True), q.plan_stats(g, p, fuse=False)
    assert fused.n_buckets == plain.n_buckets
    assert fused.alg_bytes == plain.alg_bytes and fused.sum_ops == plain.sum_ops
    assert fused.max_width == plain.max_width == max(max(q.simulate_widths(g, i, p))
                                                     for i in range(g.m))
    assert plain.n_segments == 0 and plain.dev_bytes == plain.alg_bytes
    assert fused.n_segments > 0
    # every bucket is either one device op or one stage of a segment
    assert fused.n_device_ops + fused.n_fused_ops == plain.n_device_ops
    assert fused.n_levels < plain.n_levels
    assert fused.dev_bytes < plain.dev_bytes
    # level placement differs between the two programs (ALAP over units)
    assert fused.arena_bytes <= 1.25 * plain.arena_bytes


def test_c2_fused_traffic(q, golden):
    c, p = _cfg(golden, "C2")
    g = q.random_regular(c["n"], 3, c["seed"])
    inf = q.plan_stats(g, p)
    # 19.8 GB of per-bucket bytes -> about 1 GB the fused program must move
    assert inf.alg_bytes == pytest.approx(1.977e10, rel=1e-3)
    assert inf.dev_bytes < 0.08 * inf.alg_bytes


def test_segment_shapes(q, golden):
    c, p = _cfg(golden, "C2")
    g = q.random_regular(c["n"], 3, c["seed"])
    segs = q.plan_segments(g, p)
    assert segs and len(segs) == q.plan_stats(g, p).n_segments
    levels = [s["level"] for s in segs]
    assert levels == sorted(levels)
    for s in segs:
        assert 2 <= s["L"] <= 9 and 0 <= s["cy"] <= min(s["ry"], 5)
        assert s["nops"] == sum(st[0] for st in s["stages"]) <= 16
        nt1, ns1, main1, _ = s["stages"][0]
        assert main1 == -1 and ns1 <= 1 and nt1 <= 6
        for nt, ns, main, mem in s["stages"][1:]:
            assert ns == 1 and nt <= 4 and main == nt - 1
            assert mem[main][0] == 0  # placeholder: read from registers
            assert all(rank > 0 for rank, _, _ in mem[:main])
        # stage i's result rank shrinks by its summed var: rY = r_1 - (L - 1)
        if s["rb2"] is not None:
            # quad tiles: stage 1 = [prefix..., A, B]; rb read by A alone, rb2 by B alone
            assert s["cy"] == 5 and 2 <= nt1 <= 4 and s["rb"] != s["rb2"]
            mem1 = s["stages"][0][3]
            ca, cb = 32 + s["rb"], 32 + s["rb2"]
            assert ca in mem1[-2][2] and cb not in mem1[-2][2]
            assert cb in mem1[-1][2] and ca not in mem1[-1][2]
            assert all(ca not in c and cb not in c for _, _, c in mem1[:-2])
        elif s["rb"] is not None:
            # paired rows: full lane tiles, a tile bit that no side member reads
            assert s["cy"] == 5 and 0 <= s["rb"] < s["ry"] - 5 and nt1 <= 4
            for nt, ns, main, mem in s["stages"][1:]:
                for t, (rank, _, codes) in enumerate(mem):
                    assert t == main or 32 + s["rb"] not in codes
    assert any(s["rb2"] is not None for s in segs)


def test_pairing_switch(q, golden):
    # QTNG_SEG_PAIR=0 disables paired rows, QTNG_SEG_QUAD=0 quad tiles (read
    # once per process: child)
    c, p = _cfg(golden, "C2")
    code = ("import sys; sys.path.insert(0, %r); import paper_2204_06045_b200 as q; "
            "g = q.random_regular(%d, 3, %d); "
            "print(sum(s['rb'] is not None and s['rb2'] is None for s in q.plan_segments(g, %d)), "
            "sum(s['rb2'] is not None for s in q.plan_segments(g, %d)))") % (
                ROOT, c["n"], c["seed"], p, p)
    for env, want in (({"QTNG_SEG_PAIR": "0"}, lambda pr, qd: pr == 0 and qd > 0),
                      ({"QTNG_SEG_QUAD": "0"}, lambda pr, qd: pr > 0 and qd == 0),
                      ({"QTNG_SEG_QUAD": "0", "QTNG_SEG_PAIR": "0"}, lambda pr, qd: pr == qd == 0)):
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        pr, qd = (int(x) for x in r.stdout.strip().splitlines()[-1].split())
        assert want(pr, qd), (env, pr, qd)


def _child_energy(name, env):
    code = r'''
import json, sys
sys.path.insert(0, %r)
import numpy as np
import paper_2204_06045_b200 as q
c = json.load(open(%r))["configs"][%r]
g = q.random_regular(c["n"], 3, c["seed"])
plan = q.Plan(g, len(c["gammas"]))
t = plan.execute(q.Angles(c["gammas"], c["betas"]))
inf = plan.info()
print(json.dumps({"terms": [[float(x.real), float(x.imag)] for x in t], "segments": int(inf.n_segments)}))
''' % (ROOT, os.path.join(ROOT, "tests", "golden", "energies.json"), name)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C2", "C4"])
def test_fused_equals_unfused_bitwise(golden, name):
    ref = np.array([complex(x, y) for x, y in golden["configs"][name]["terms_naive"]])
    plain = _child_energy(name, {"QTNG_FUSE": "0"})
    assert plain["segments"] == 0
    for env in ({"QTNG_SEG_J": "1"}, {"QTNG_SEG_J": "3"}, {"QTNG_SEG_J": "8"},
                {"QTNG_SEG_PAIR": "0"}, {"QTNG_SEG_PAIR": "1"}, {"QTNG_SEG_PAIR_NT": "2"},
                {"QTNG_SEG_QUAD": "0"}, {"QTNG_SEG_QUAD": "1"},
                {"QTNG_SEG_QUAD": "1", "QTNG_SEG_J": "2"},
                {"QTNG_SEG_QUAD": "0", "QTNG_SEG_PAIR": "0"},
                {"QTNG_LEVELS": "0"}, {"QTNG_LEVELS": "1"}, {"QTNG_SEG_STARVED": "1024"}):
        fused = _child_energy(name, env)
        assert fused["segments"] > 0
        assert fused["terms"] == plain["terms"], str(env)
    got = np.array([complex(x, y) for x, y in plain["terms"]])
    assert np.array_equal(got, ref)


@pytest.mark.gpu
def test_flow_executor_bitwise(golden):
    # the experimental single-kernel dataflow executor (QTNG_FLOW=1) runs the
    # same units: terms identical to the level-synchronous program's
    ref = [[x, y] for x, y in golden["configs"]["C2"]["terms_naive"]]
    flow = _child_energy("C2", {"QTNG_FLOW": "1"})
    assert flow["terms"] == ref
