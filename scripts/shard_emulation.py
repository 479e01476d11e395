"""The distributed plan on ONE GPU: G in-process shards (one host thread
each, one device) running the same schedule, block-split sweeps and in-place
pipelined remaps as G GPUs would, the remap swaps going through HBM instead
of NVLink.  Reports per-run wall time against the dense engine and the
remap records ('W' pipelined: the block-split group-A sweep with its swaps,
'T' serial exchange, 'Y' fused).

    python scripts/shard_emulation.py [n p prec G ...]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_26423_b200 as L  # noqa: E402
from paper_2604_26423_b200 import _native  # noqa: E402


def main():
    args = sys.argv[1:] or ["33", "3", "fp64", "2", "4", "8"]
    n, p, prec = int(args[0]), int(args[1]), args[2]
    Gs = [int(g) for g in args[3:]]
    inst = L.generate_instance(n, 1)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=p))
    B = 8 if prec == "fp32" else 16
    out = {"n": n, "p": p, "precision": prec, "state_GiB": (B << n) / 2**30, "runs": {}}
    # dense reference: the same circuit as one state
    for rep in range(2):
        t0 = time.perf_counter()
        sv = L.run_circuit(circ, prec, memory_budget=1 << 40)
        sv.norm_squared()
        dense_s = time.perf_counter() - t0
        sv.release()
    _native.drain_pool()
    out["dense_wall_ms"] = dense_s * 1e3
    for G in Gs:
        plan = L.plan_for_shard_count(n, G)
        for rep in range(2):
            t0 = time.perf_counter()
            sv, rec = L.run_circuit_sharded(circ, plan, prec, memory_budget=1 << 40, devices=[0])
            sv.norm_squared()
            wall = time.perf_counter() - t0
            mode = getattr(sv, "remap_mode", None)
            sv.release()
        kinds = "".join(g.kind for g in rec.gates)
        remaps = [g for g in rec.gates if g.kind in "WTY"]
        moved = sum(g.amps_exchanged for g in remaps) * B
        out["runs"][G] = {
            "wall_ms": wall * 1e3, "device_compute_ms": rec.compute_seconds * 1e3,
            "remap_records_ms": [round(g.exchange_s * 1e3, 3) for g in remaps], "kinds": kinds,
            "remap_bytes_per_run": moved, "transport": mode,
            "vs_dense": wall / dense_s,
        }
        print(json.dumps({G: out["runs"][G]}), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
