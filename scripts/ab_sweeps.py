"""A/B timing of two builds of liblrq on the same GPU: per sweep label
(P/M/F/R on groups A/H/H4) mean CUDA-event ms of one n, p run, alternating
the builds over several processes so clock drift hits both alike.

    python scripts/ab_sweeps.py OLD.so NEW.so [n p prec rounds]

A build may carry environment settings: "lib.so|LRQ_WD_QUARTER=0".
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
sys.path.insert(0, %r)
import paper_2604_26423_b200 as L
from paper_2604_26423_b200 import _native
sys.path.insert(0, %r)
from bench import sweep_labels
n, p, prec = %d, %d, %r
inst = L.generate_instance(n, 1)
lay = L.lower_circuit(L.build_circuit(inst, L.LrQaoaParams(p=p)))
B = 8 if prec == "fp32" else 16
dev = _native.DeviceState(n, B)
dev.set_cost(inst.weights())
dev.set_timing(True)
out = {}
for rep in range(3):
    dev.run(lay.phase, lay.mixer)
    ms, kinds = dev.timings()
    if rep == 0:
        continue
    labels = sweep_labels(n, B, p, 1)
    sweeps = [m for m, k in zip(ms, kinds) if k in "PMFRLQ"]
    for (lab, _), m in zip(labels, sweeps):
        out.setdefault(lab, []).append(m)
print(json.dumps(out))
"""


def run(lib, n, p, prec):
    # "path|KEY=VAL|KEY2=VAL2": the build plus environment settings
    lib, *assigns = lib.split("|")
    env = dict(os.environ, LRQ_LIB=lib)
    env.update(a.split("=", 1) for a in assigns)
    code = CHILD % (ROOT, ROOT, n, p, prec)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"{lib} {assigns}: {r.stderr[-800:]}")
    return json.loads(r.stdout.strip().splitlines()[-1])


def main():
    old, new = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    p = int(sys.argv[4]) if len(sys.argv) > 4 else 10
    prec = sys.argv[5] if len(sys.argv) > 5 else "fp32"
    rounds = int(sys.argv[6]) if len(sys.argv) > 6 else 4
    acc = {"old": {}, "new": {}}
    for _ in range(rounds):
        for tag, lib in (("old", old), ("new", new)):
            for k, v in run(lib, n, p, prec).items():
                acc[tag].setdefault(k, []).extend(v)
    print(f"# ab_sweeps n={n} p={p} {prec}, {rounds} alternating processes per build; mean ms (min)")
    for k in acc["old"]:
        o, w = acc["old"][k], acc["new"].get(k, [])
        mo, mw = sum(o) / len(o), sum(w) / len(w)
        print(f"{k:8s} old {mo:8.3f} ({min(o):.3f})  new {mw:8.3f} ({min(w):.3f})  {100 * (mw / mo - 1):+6.2f}%  n={len(o)}")
    to = sum(sum(v) for v in acc["old"].values()) / (2 * rounds)
    tn = sum(sum(v) for v in acc["new"].values()) / (2 * rounds)
    print(f"per-run sweep total: old {to:.2f} ms, new {tn:.2f} ms ({100 * (tn / to - 1):+.2f}%)")


if __name__ == "__main__":
    main()
