#!/usr/bin/env python3
"""Generate the committed golden fixtures under tests/golden/ from the
UNMODIFIED reference (oracle/_ref/libqtnsim_ref.so).  TEST INFRASTRUCTURE ONLY.

Run here (where /root/reference exists):  make -C oracle && python oracle/gen_golden.py

Every float is stored with 17 significant digits (round-trip exact), so the
GPU path can be checked bit-for-bit against the reference's naive backend.

Fingerprint recipe (FNV-1a 64 over int64 little-endian values):
  graph_edges      u, v for every edge (sorted edge list)
  elim_orders      per edge: the greedy_order ids (= the unmerged buckets'
                   sum vars, assign_buckets ordering.cpp:44-68), then -1
  initial_buckets  per edge, per bucket: sum vars, -2, each tensor's vars
                   followed by -3, then -4
  simulated_widths per edge: simulate_widths (engine.cpp:235-240), then -5
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")

CONFIGS = {
    # C1 = calibration trial graph, C2 = acceptance scale run
    # (proj/tests/acceptance.cpp:70-71), C4 = N=100 p=3 seed 1.
    "C1": dict(n=10, d=3, seed=7, gammas=[0.4], betas=[0.3]),
    "C2": dict(n=30, d=3, seed=104478, gammas=[0.30, 0.25, 0.20, 0.15],
               betas=[0.35, 0.30, 0.25, 0.20]),
    "C4": dict(n=100, d=3, seed=1, gammas=[0.30, 0.25, 0.20], betas=[0.35, 0.30, 0.25]),
}


def f17(x: float) -> float:
    return float("%.17g" % x)


def schedules(n, edges, g, b, merged=False):
    for i in range(len(edges)):
        ints, data, nb = O.ref_edge_schedule(n, edges, g, b, i, merged)
        yield i, O.parse_schedule(ints, nb)


def fingerprints(n, edges, g, b):
    order, init, widths = [], [], []
    n_buckets = 0
    shapes = []
    for i, sched in schedules(n, edges, g, b):
        n_buckets += len(sched)
        for sums, ts in sched:
            order += sums
            init += sums + [-2]
            for t in ts:
                init += t + [-3]
            init += [-4]
        order.append(-1)
        w = [int(x) for x in O.ref_simulate_widths(n, edges, g, b, i)]
        widths += w + [-5]
        shapes.append(w)
    return dict(graph_edges="%016x" % O.fnv1a_int64(np.asarray(edges).reshape(-1)),
                elim_orders="%016x" % O.fnv1a_int64(order),
                initial_buckets="%016x" % O.fnv1a_int64(init),
                simulated_widths="%016x" % O.fnv1a_int64(widths),
                n_buckets=n_buckets), shapes


def instance_record(name, n, seed, gammas, betas, jobs=8, sv=True, widths=False):
    t0 = time.time()
    edges = O.ref_random_regular(n, 3, seed)
    naive, _ = O.ref_edge_terms(n, edges, gammas, betas, "naive", jobs=jobs)
    matmul, _ = O.ref_edge_terms(n, edges, gammas, betas, "matmul", jobs=jobs)
    e_naive, _, nrec, peak = O.ref_energy(n, edges, gammas, betas, "naive", jobs=jobs)
    e_matmul, _, _, _ = O.ref_energy(n, edges, gammas, betas, "matmul", jobs=jobs)
    fp, shapes = fingerprints(n, edges, gammas, betas)
    rec = dict(name=name, n=n, d=3, seed=seed, gammas=[f17(x) for x in gammas],
               betas=[f17(x) for x in betas], edges=edges.tolist(),
               energy_naive=f17(e_naive), energy_matmul=f17(e_matmul),
               terms_naive=[[f17(z.real), f17(z.imag)] for z in naive],
               terms_matmul=[[f17(z.real), f17(z.imag)] for z in matmul],
               n_records=int(nrec), peak_tensor_bytes=int(peak),
               max_width=max(max(s) for s in shapes), fingerprints=fp)
    if widths:
        rec["simulated_widths"] = shapes
    if sv and n <= 20:
        rec["energy_statevector"] = f17(O.ref_statevector_energy(n, edges, gammas, betas))
    if n <= 16:
        e_merged, _, _, _ = O.ref_energy(n, edges, gammas, betas, "matmul", merged=True,
                                         jobs=jobs)
        rec["energy_merged"] = f17(e_merged)
    print(f"  {name}: E={e_naive!r} buckets={fp['n_buckets']} ({time.time() - t0:.1f}s)",
          flush=True)
    return rec


def acceptance_instances():
    lib = O.ref_lib()
    lib.ref_acceptance_instances.argtypes = [np.ctypeslib.ndpointer(np.int32),
                                             np.ctypeslib.ndpointer(np.uint64),
                                             np.ctypeslib.ndpointer(np.int32),
                                             np.ctypeslib.ndpointer(np.float64)]
    ns = np.zeros(20, np.int32)
    seeds = np.zeros(20, np.uint64)
    ps = np.zeros(20, np.int32)
    ang = np.zeros(120, np.float64)
    k = lib.ref_acceptance_instances(ns, seeds, ps, ang)
    out = []
    for i in range(k):
        p = int(ps[i])
        out.append((int(ns[i]), int(seeds[i]), list(ang[i * 6:i * 6 + p]),
                    list(ang[i * 6 + 3:i * 6 + 3 + p])))
    return out


def random_buckets(seed=2204, count=48):
    """Random buckets in the style of proj/tests/test_engine.cpp:48-65: the
    first tensor carries every var, others a random subset, axis order
    shuffled; plus rank-0/duplicate-free edge cases."""
    rng = np.random.default_rng(seed)
    out = []
    for trial in range(count):
        n_t = 1 + trial % 6
        n_vars = 2 + trial % 9
        n_sum = 1 + trial % 3 if trial % 7 else 0
        n_sum = min(n_sum, n_vars)
        base = rng.choice(np.arange(0, 40), size=n_vars, replace=False)
        ts = []
        for t in range(n_t):
            vs = [int(v) for v in base if t == 0 or rng.integers(2)]
            if not vs:
                vs = [int(base[rng.integers(n_vars)])]
            rng.shuffle(vs)
            d = rng.uniform(-1, 1, 1 << len(vs)) + 1j * rng.uniform(-1, 1, 1 << len(vs))
            ts.append((vs, d))
        sums = sorted(int(v) for v in rng.choice(base, size=n_sum, replace=False))
        ov, naive = O.ref_contract_bucket(ts, sums, "naive")
        mv, matmul = O.ref_contract_bucket(ts, sums, "matmul")
        out.append(dict(
            tensors=[dict(vars=v, re=[f17(x) for x in d.real], im=[f17(x) for x in d.imag])
                     for v, d in ts],
            # matmul_vars can differ from out_vars: MatmulBackend returns a lone
            # tensor with no present sum var unpermuted (contraction.cpp:124),
            # breaking the ascending-axes contract of engine.hpp:28-29.
            sum_vars=sums, out_vars=ov, matmul_vars=mv,
            naive_re=[f17(x) for x in naive.real], naive_im=[f17(x) for x in naive.imag],
            matmul_re=[f17(x) for x in matmul.real], matmul_im=[f17(x) for x in matmul.imag]))
    # known answers from test_engine.cpp:77-89 (<+|+> = 1)
    r = 1.0 / np.sqrt(2.0)
    ts = [([0], np.array([r, r], complex)), ([0], np.array([r, r], complex))]
    ov, naive = O.ref_contract_bucket(ts, [0], "naive")
    out.append(dict(tensors=[dict(vars=v, re=list(d.real), im=list(d.imag)) for v, d in ts],
                    sum_vars=[0], out_vars=ov, matmul_vars=ov, naive_re=list(naive.real),
                    naive_im=list(naive.imag), matmul_re=list(naive.real),
                    matmul_im=list(naive.imag)))
    return out


def refusals():
    out = []
    # C1 with a tiny cap: the refusal surfaces as ScheduleError naming the edge
    # (engine.cpp:160-169 wrapped at engine.cpp:543-546).
    for name, n, seed, g, b, cap in [("C1_cap3", 10, 7, [0.4], [0.3], 3),
                                     ("N50p5_cap14", 50, 1, [0.3] * 5, [0.2] * 5, 14)]:
        edges = O.ref_random_regular(n, 3, seed)
        try:
            O.ref_energy(n, edges, g, b, "naive", max_width=cap, jobs=8)
            code, msg = 0, ""
        except O.OracleError as ex:
            code, msg = ex.code, str(ex)
        out.append(dict(name=name, n=n, seed=seed, gammas=g, betas=b, max_width=cap,
                        code=code, message=msg))
        print(f"  refusal {name}: {code} {msg}")
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    if "--buckets-only" in sys.argv:
        with open(os.path.join(OUT, "buckets.json"), "w") as f:
            json.dump(random_buckets(), f)
        return
    print("configs:")
    cfgs = {}
    for name, c in CONFIGS.items():
        cfgs[name] = instance_record(name, c["n"], c["seed"], c["gammas"], c["betas"],
                                     widths=(name != "C4"))
    print("acceptance instances:")
    acc = [instance_record(f"acc{i}", n, s, g, b)
           for i, (n, s, g, b) in enumerate(acceptance_instances())]
    with open(os.path.join(OUT, "energies.json"), "w") as f:
        json.dump(dict(configs=cfgs, acceptance=acc, refusals=refusals()), f)
    # full schedules of C1 (small) for structural comparison
    c = CONFIGS["C1"]
    edges = O.ref_random_regular(c["n"], 3, c["seed"])
    sch = [dict(edge=edges[i].tolist(), buckets=[dict(sum_vars=s, tensors=t) for s, t in sc])
           for i, sc in schedules(c["n"], edges, c["gammas"], c["betas"])]
    with open(os.path.join(OUT, "schedule_C1.json"), "w") as f:
        json.dump(sch, f)
    with open(os.path.join(OUT, "buckets.json"), "w") as f:
        json.dump(random_buckets(), f)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
