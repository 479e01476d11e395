"""Per-config measurements on one B200 (BASELINE.json configs that fit one GPU).

    python scripts/bench_configs.py > profiles/r01_configs.json

For each config: device time per run (CUDA events on the engine stream, best
of `reps` after a warm-up run), layer amplitude-updates/s, per-sweep-kind
mean ms and HBM fraction (algorithmic 2 * 2^n * B bytes per sweep, P
write-only), and the exact r against C* (GPU exhaustive search).
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_26423_b200 as L  # noqa: E402
from paper_2604_26423_b200 import _native  # noqa: E402

PEAK = 6541.5
CONFIGS = [
    ("configs[0]: n=12 p=3 complex128", 12, 3, "fp64", 7),
    ("configs[1]: n=26 p=3 complex128", 26, 3, "fp64", 1),
    ("configs[2]: n=32 p=10 complex64", 32, 10, "fp32", 1),
    ("configs[3] 1-GPU point: n=33 p=3 complex128 (128 GiB)", 33, 3, "fp64", 1),
    ("n=34 p=3 complex64 (128 GiB)", 34, 3, "fp32", 1),
]


def run(label, n, p, prec, seed, reps=3):
    pb = 16 if prec == "fp64" else 8
    inst = L.generate_instance(n, seed)
    lay = L.lower_circuit(L.build_circuit(inst, L.LrQaoaParams(p=p)))
    dev = _native.DeviceState(n, pb)
    dev.set_cost(inst.weights())
    dev.set_timing(True)
    best, kinds_ms = None, None
    for _ in range(reps + 1):
        dev.run(lay.phase, lay.mixer)
        ms, kinds = dev.timings()
        tot = sum(ms)
        if best is None or tot < best:
            best, kinds_ms = tot, (ms, kinds)
    red = dev.reduce()
    dev.close(park=False)
    _native.drain_pool()
    z = int(red.argmax_cut)
    cstar = float(L.cut_values(inst, [z])[0])
    ms, kinds = kinds_ms
    per = {}
    for m, k in zip(ms, kinds):
        if k in "PMFRQ":
            per.setdefault(k, []).append(m)
    sweeps = {k: {"count": len(v), "mean_ms": round(statistics.mean(v), 3),
                  "hbm_frac": round((1 if k == "P" else 2) * (pb << n) / (statistics.mean(v) * 1e-3) / 1e9 / PEAK, 3)}
              for k, v in per.items()}
    return {"config": label, "n": n, "p": p, "precision": prec, "ms_per_run": round(best, 3),
            "ms_per_layer": round(best / p, 3), "layer_amp_updates_per_s": (1 << n) * p / (best * 1e-3),
            "sweeps": sweeps, "exact_r": float(red.sum_p_cut) / cstar, "max_cut": cstar, "sum_p": red.sum_p}


def run_sharded(n, p, prec, G, seed=1):
    """The distributed plan on ONE GPU: G shard states of an in-process shard
    group (remaps are device-side block swaps in HBM instead of NCCL).  This
    measures the multi-GPU engine's per-shard sweep schedule, not NVLink."""
    inst = L.generate_instance(n, seed)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=p))
    plan = L.plan_for_shard_count(n, G)
    best, rec_best = None, None
    for _ in range(2):
        sv, rec = L.run_circuit_sharded(circ, plan, prec)
        sv.release()
        if best is None or rec.wall_seconds < best:
            best, rec_best = rec.wall_seconds, rec
    sweeps = {}
    for g in rec_best.gates:
        sweeps.setdefault(g.kind, []).append(g.compute_s + g.exchange_s)
    return {"config": f"sharded on one GPU: n={n} p={p} {prec} G={G}", "n": n, "p": p, "precision": prec,
            "shards": G, "wall_s": round(best, 4),
            "device_ms_per_shard_launch": {k: round(1e3 * statistics.mean(v), 3) for k, v in sweeps.items()},
            "amps_exchanged": rec_best.amps_exchanged}


def main():
    out = []
    for cfg in CONFIGS:
        t0 = time.time()
        r = run(*cfg)
        r["wall_s"] = round(time.time() - t0, 1)
        out.append(r)
        print(json.dumps(r), file=sys.stderr, flush=True)
    for G in (2, 4, 8):
        r = run_sharded(30, 3, "fp32", G)
        out.append(r)
        print(json.dumps(r), file=sys.stderr, flush=True)
    print(json.dumps({"device": "1x B200", "peak_hbm_gbs": PEAK, "results": out}, indent=1))


if __name__ == "__main__":
    main()
