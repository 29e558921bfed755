#!/usr/bin/env python3
"""Parity of every build/variants/*.so on C1/C2 (debug aid for kernel variants)."""
import glob, os, subprocess, sys, json
ROOT='/root/repo'
code = r'''
import sys, json; sys.path.insert(0, %r)
import numpy as np, paper_2204_06045_b200 as q
c = json.load(open(%r))["configs"]
for name in ("C1", "C2"):
    cc = c[name]; g = q.random_regular(cc["n"], 3, cc["seed"])
    plan = q.Plan(g, len(cc["gammas"]))
    try:
        t = plan._raw_execute(q.Angles(cc["gammas"], cc["betas"])) if hasattr(plan, "_raw_execute") else plan.execute(q.Angles(cc["gammas"], cc["betas"]))
        e = 0.5*g.m - 0.5*float(np.sum(t.real)); print(name, e, e == cc["energy_naive"])
    except Exception as ex: print(name, repr(ex)[:100])
''' % (ROOT, ROOT + "/tests/golden/energies.json")
for so in sorted(glob.glob(ROOT + "/build/variants/*.so")):
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, QTNG_LIB_PATH=so), capture_output=True, text=True, timeout=300)
    print(os.path.basename(so), r.stdout.strip(), r.stderr[-300:])
