"""Quick per-sweep timing probe (CUDA events on the engine stream)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2604_26423_b200 as L  # noqa: E402
from paper_2604_26423_b200 import _native  # noqa: E402

PEAK = 6541.5


def probe(n, p, prec, reps=2):
    inst = L.generate_instance(n, 1)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=p))
    lay = L.lower_circuit(circ)
    pb = 8 if prec == "fp32" else 16
    dev = _native.DeviceState(n, pb)
    dev.set_cost(inst.weights())
    dev.set_timing(True)
    for r in range(reps):
        t0 = time.perf_counter()
        dev.run(lay.phase, lay.mixer)
        wall = time.perf_counter() - t0
    ms, kinds = dev.timings()
    byts = 2 * (1 << n) * pb
    print(f"n={n} p={p} {prec}: wall {wall*1e3:.1f} ms, device sum {sum(ms):.1f} ms, launches {len(ms)}")
    for m, k in zip(ms, kinds):
        bw = (byts if k != 'P' or True else byts) / (m * 1e-3) / 1e9
        print(f"   {k} {m:8.3f} ms  {bw:8.1f} GB/s  ({bw/PEAK*100:5.1f}% of measured)")
    red = dev.reduce()
    print("   sum_p", red.sum_p, "sum_pC", red.sum_p_cut)
    dev.close()


if __name__ == "__main__":
    for spec in sys.argv[1:]:
        n, p, prec = spec.split(",")
        probe(int(n), int(p), prec)
