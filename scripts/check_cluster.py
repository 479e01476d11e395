"""Cluster-pair sweeps (complex64 C groups) against the single-CTA plan of
the same circuit: normwise amplitude difference, r, and per-sweep times.

    python scripts/check_cluster.py 24,2 29,3 32,10
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_26423_b200 as L  # noqa: E402
from paper_2604_26423_b200 import _native  # noqa: E402


def run(n, p, cluster, dbeta=0.2):
    os.environ["LRQ_CLUSTER"] = "1" if cluster else "0"
    inst = L.generate_instance(n, 1)
    lay = L.lower_circuit(L.build_circuit(inst, L.LrQaoaParams(p=p, delta_beta=dbeta)))
    dev = _native.DeviceState(n, 8)
    dev.set_cost(inst.weights())
    dev.run(lay.phase, lay.mixer)
    dev.set_timing(True)
    dev.run(lay.phase, lay.mixer)
    ms, kinds = dev.timings()
    red = dev.reduce()
    probe = np.concatenate([dev.copy_amps(0, 1 << 16), dev.copy_amps((1 << n) - (1 << 16), 1 << 16),
                            dev.copy_amps(1 << (n - 1), 1 << 16)])
    full = dev.copy_amps() if n <= 28 else None
    dev.close(park=False)
    plan = json.loads(_native.describe_plan(n, 8, p))
    labels = [f"{s['kind']}({plan['groups'][s['group']]['kind']})" for s in plan["sweeps"]]
    return red, probe, full, list(zip(labels, [round(m, 3) for m, k in zip(ms, kinds) if k in "PMFRQ"]))


for arg in sys.argv[1:] or ["29,3"]:
    parts = arg.split(",")
    n, p = int(parts[0]), int(parts[1])
    dbeta = float(parts[2]) if len(parts) > 2 else 0.2
    a = run(n, p, True, dbeta)
    b = run(n, p, False, dbeta)
    d = np.linalg.norm(a[1].astype(np.complex128) - b[1]) / np.linalg.norm(b[1])
    out = {"n": n, "p": p, "dbeta": dbeta, "probe_normwise": float(d),
           "sum_p": [a[0].sum_p, b[0].sum_p], "sum_p_cut": [a[0].sum_p_cut, b[0].sum_p_cut],
           "cluster_sweeps": a[3], "plain_sweeps": b[3]}
    if a[2] is not None:
        out["full_normwise"] = float(np.linalg.norm(a[2].astype(np.complex128) - b[2]) / np.linalg.norm(b[2]))
    print(json.dumps(out), flush=True)
