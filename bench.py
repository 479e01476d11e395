"""Benchmark of the LR-QAOA state-vector hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 1..5] [--n N --p P --precision fp32|fp64 --shots S]

Workloads (BASELINE.json configs, fully connected weighted MaxCut LR-QAOA,
instance generate_instance(n, 1), ramp 0.2/0.2):
  N = 1 (default): configs[2], n=32, p=10, complex64 (32 GiB state), 1k shots.
        The same line also carries configs[1] (n=26 p=3 complex128) and the
        one-GPU point of configs[3] (n=33 p=3 complex128, 128 GiB) under
        "configs", measured on the device the same way.
  N > 1 (default): one distributed state of n = 33 + log2(N) qubits,
        complex128, p=3, 10k shots - configs[3] at N=2 (n=34) and configs[4]
        at N=8 (n=36), 2^33 amplitudes (128 GiB) per GPU (weak scaling).
  --config k picks BASELINE configs[k-1] explicitly (configs 4/5 at N=1 fall
        back to the largest one-GPU size, n=33).
One step = the whole hot path on one batch: H layer + p layers (fused
sweeps, remaps between GPUs) + fused final pass (sum p, sum pC, min/max E,
CDF block sums) + inverse-CDF samples.

value     layer amplitude-updates/s = 2^n * p * steps / device time (device
          time = max over ranks of CUDA events on the engine stream).
e2e       the same metric through the public drop-in API (run_circuit /
          run_circuit_distributed -> exact_expected_r -> sample), host inputs
          and outputs inside the timed region.
roofline  the dominant kernel (largest share of the step): algorithmic bytes
          per launch (2 * 2^n_loc * B; the write-only first sweep 2^n_loc * B)
          / its mean CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs;
          "per_kernel" lists every sweep kind (P/M/F/R on groups A/H/H4).
cpu_baseline  the reference's own CPU engine (baseline/_ref lrqbench if
          installed, else the oracle port): run_circuit_sharded with one
          thread per shard on all host cores over a bounded gate sample,
          extrapolated per gate to the workload; single-thread run_circuit
          beside it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
METRIC = "LR-QAOA layer amplitude-updates/s"
sys.path.insert(0, ROOT)

# BASELINE.json configs: (n, p, precision, shots)
CONFIGS = {1: (12, 3, "fp64", 1000), 2: (26, 3, "fp64", 1000), 3: (32, 10, "fp32", 1000),
           4: (34, 3, "fp64", 10000), 5: (36, 3, "fp64", 10000)}
BUDGET = 1 << 40  # explicit memory budget (the reference's default is 4 GiB)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=0, choices=[0, 1, 2, 3, 4, 5])
    ap.add_argument("--n", type=int, default=0, help="override: total qubits")
    ap.add_argument("--p", type=int, default=0)
    ap.add_argument("--precision", default="", choices=["", "fp32", "fp64"])
    ap.add_argument("--shots", type=int, default=0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="budget of the CPU reference sample")
    ap.add_argument("--no-extra-configs", action="store_true", help="N=1: skip the embedded configs 2 and 4")
    return ap.parse_args()


def workload(args, world):
    """(n_total, p, precision, shots, label, scaling) of this run."""
    g = world.bit_length() - 1
    cfg = args.config
    if cfg == 0:
        cfg = 3 if world == 1 else 45
    if cfg == 45:  # default multi-GPU family: 2^33 complex128 amplitudes per GPU
        n, p, prec, shots = 33 + g, 3, "fp64", 10000
        label = (f"LR-QAOA p=3, n={n} fully connected weighted MaxCut, complex128 over {world} B200s "
                 f"(2^33 amplitudes per GPU; BASELINE configs[3] at N=2, configs[4] at N=8)")
        scaling = "weak"
    else:
        n, p, prec, shots = CONFIGS[cfg]
        if cfg in (4, 5) and n - g > 33:
            n = 33 + g  # the state does not fit: the largest size this GPU count holds
        if cfg == 3 and world > 1:
            n = 32 + g  # weak scaling of the one-GPU workload
        label = (f"LR-QAOA p={p}, n={n} fully connected weighted MaxCut, "
                 f"{'complex64' if prec == 'fp32' else 'complex128'} on {world}xB200 (BASELINE configs[{cfg - 1}]"
                 + (f", n reduced from {CONFIGS[cfg][0]} to fit" if n != CONFIGS[cfg][0] and cfg != 3 else "") + ")")
        scaling = "strong" if cfg in (4, 5) and world > 1 and n == CONFIGS[cfg][0] else "weak"
    if args.n or args.p or args.precision:
        n = args.n + (g if world > 1 else 0) if args.n else n
        p = args.p or p
        prec = args.precision or prec
        label = (f"LR-QAOA p={p}, n={n} fully connected weighted MaxCut, "
                 f"{'complex64' if prec == 'fp32' else 'complex128'} on {world}xB200 (custom size)")
    shots = args.shots or shots
    return n, p, prec, shots, label, scaling


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def init_dist(world):
    if world <= 1:
        return None
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    return dist


def max_over_ranks(dist, x: float) -> float:
    if dist is None:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def profiled_traffic():
    """dram read+write bytes per launch by sweep label, from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


# ---------------------------------------------------------------------------
# per-kernel roofline


def sweep_labels(n_local, B, p, world):
    """Label of every sweep record of one run, in launch order: kind(group),
    e.g. F(H), M(A), R(A), and the kernel that runs it."""
    from paper_2604_26423_b200 import _native

    if world > 1:
        plan = json.loads(_native.describe_dist_plan(n_local + (world.bit_length() - 1), world.bit_length() - 1, B, p))
    else:
        plan = json.loads(_native.describe_plan(n_local, B, p))
    out = []
    for sw in plan["sweeps"]:
        gk = plan["groups"][sw["group"]]["kind"]
        if sw.get("prog") == 1:
            kern = "sweep_wd_kernel"
        elif B == 8 and gk != "A" and sw["kind"] in "MF":
            kern = "sweep_tma_kernel"
        else:
            kern = "sweep_kernel"
        out.append((f"{sw['kind']}({gk})", kern))
    return out


def per_kernel(ms, kinds, labels, n_local, B, peak, steps):
    """Group the sweep records of `steps` runs by label: mean ms, bytes, GB/s,
    fraction of peak, share of the sweeps' time.  Records other than sweeps
    (remaps, flips, the finalize) are skipped; sweeps map onto `labels` (one
    run's plan) in order."""
    recs = {}
    j = 0
    for m, k in zip(ms, kinds):
        if k in "PMFRQ":
            lab, kern = labels[j % len(labels)]
            j += 1
            recs.setdefault(lab, {"kernel": kern, "ms": []})["ms"].append(m)
    total = sum(sum(r["ms"]) for r in recs.values()) or 1.0
    out = {}
    for lab, r in recs.items():
        byts = (1 if lab.startswith("P") or lab.startswith("Q") else 2) * (B << n_local)  # P writes, Q reads only
        avg = statistics.mean(r["ms"])
        gbs = byts / (avg * 1e-3) / 1e9
        out[lab] = {"kernel": r["kernel"], "launches_per_step": len(r["ms"]) // max(1, steps), "ms_avg": round(avg, 4),
                    "bytes_per_launch": byts, "achieved_GBps": round(gbs, 1), "frac": round(gbs / peak, 4),
                    "time_share": round(sum(r["ms"]) / total, 4)}
    return out


def dominant(pk, peak):
    """The kernel function with the largest share of the sweep time, with its
    achieved bandwidth over all its launches (sum of bytes / sum of time)."""
    by = {}
    for lab, v in pk.items():
        d = by.setdefault(v["kernel"], {"labels": [], "bytes": 0.0, "ms": 0.0, "share": 0.0})
        d["labels"].append(lab)
        d["bytes"] += v["bytes_per_launch"] * v["launches_per_step"]
        d["ms"] += v["ms_avg"] * v["launches_per_step"]
        d["share"] += v["time_share"]
    k = max(by, key=lambda x: by[x]["share"])
    d = by[k]
    gbs = d["bytes"] / (d["ms"] * 1e-3) / 1e9
    n_launch = sum(pk[lab]["launches_per_step"] for lab in d["labels"])
    return k, {"labels": sorted(d["labels"]), "achieved": round(gbs, 1), "frac": round(gbs / peak, 4),
               "time_share": round(d["share"], 4), "launches_per_step": n_launch,
               "bytes_per_launch_avg": d["bytes"] / max(1, n_launch), "launch_ms_avg": d["ms"] / max(1, n_launch)}


def kernel_launches(kinds, n_local, tile_bits=13):
    """Our kernel launches behind the engine's timing records: one per sweep
    ('P','M','F','R','Q'), three for the multi-CTA finalize ('Z', tile count
    >= 8192), two for a deferred-flip reversal ('X'); remaps are swap kernels
    over peer memory ('W', 'T': world-1 per remap, counted by the caller) or
    the preceding sweep's own stores ('Y': none)."""
    z = 3 if (1 << max(0, n_local - tile_bits)) >= 8192 else 1
    return sum(z if k == "Z" else 2 if k == "X" else 0 if k in "TYW" else 1 for k in kinds)


# ---------------------------------------------------------------------------
# CPU reference: the reference package's own engine on the host cores


def _reference_module():
    """lrqbench from baseline/_ref (the unmodified reference, pip-installed
    there); None if it is not installed."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "lrqbench")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import lrqbench  # noqa: F401

        return lrqbench
    except ImportError:
        return None


def cpu_reference(n, p, precision, budget_s, seed):
    """Time the reference's CPU engine on a bounded sample of the workload.

    Threaded: lrqbench.run_circuit_sharded (one thread per shard, the
    reference's own parallel engine) on the H layer, a stride sample of
    layer 0's RZZ gates and its RX gates at n_run <= n qubits; per-gate cost
    is linear in 2^n (memory-bound numpy passes), so
    t_layer(n) = (E_n * t_RZZ + n * t_RX) * 2^(n - n_run).
    Single thread: lrqbench.run_circuit (engine.py:198-207) on a prefix of
    the same gates.  Without baseline/_ref, the oracle port does the same."""
    import psutil

    R = _reference_module()
    cores = len(os.sched_getaffinity(0))
    B = 8 if precision == "fp32" else 16
    avail = psutil.virtual_memory().available
    n_run = min(n, 28 if B == 8 else 27)
    while n_run > 12 and 4 * (B << n_run) > 0.5 * avail:
        n_run -= 1
    G = 1
    while G * 2 <= cores and G * 2 <= (1 << (n_run - 2)):
        G *= 2
    scale = float(1 << (n - n_run))
    E = n * (n - 1) // 2
    if R is None:
        from oracle import lrq_oracle as O

        eng = O.DenseOracle(n_run, precision, threads=cores)
        eng.amps[:] = eng.dtype.type(1.0 / np.sqrt(1 << n_run))
        w = O.instance_weights(n_run, seed)
        betas, gammas = O.ramp(p)
        pairs = O.edge_pairs(n_run)
        t_rzz, t_rx = [], []
        t0 = time.perf_counter()
        k = 0
        while time.perf_counter() - t0 < budget_s or len(t_rx) < 2:
            a, b = pairs[(7 * k) % len(pairs)]
            s = time.perf_counter()
            eng.rzz(a, b, 2.0 * gammas[0] * w[(7 * k) % len(pairs)])
            t_rzz.append(time.perf_counter() - s)
            if k % 3 == 0:
                s = time.perf_counter()
                eng.rx(k % n_run, -2.0 * betas[0])
                t_rx.append(time.perf_counter() - s)
            k += 1
        eng.close()
        t_layer = (E * float(np.median(t_rzz)) + n * float(np.median(t_rx))) * scale
        return {"value": (1 << n) / t_layer, "unit": "amp-updates/s", "cores": cores, "kind": "port",
                "sample": f"{len(t_rzz)} RZZ + {len(t_rx)} RX gates of the oracle port of the reference's per-gate "
                          f"engine at n={n_run}, {cores} threads, x{int(scale)} to n={n}",
                "t_layer_s": t_layer, "single_thread": None}
    inst = R.generate_instance(n_run, seed)
    circ = R.build_circuit(inst, R.LrQaoaParams(p=p))
    E_run = n_run * (n_run - 1) // 2
    layer0 = circ.gates[n_run:n_run + E_run + n_run]
    rzz = [g for g in layer0 if g.kind == "RZZ"]
    rx = [g for g in layer0 if g.kind == "RX"]
    hs = circ.gates[:n_run]
    # threaded engine: size the RZZ stride sample to the time budget with a probe
    probe = R.CircuitIR(num_qubits=n_run, gates=hs[:2] + rzz[:2])
    plan = R.plan_for_shard_count(n_run, G)
    t0 = time.perf_counter()
    R.run_circuit_sharded(probe, plan, precision, memory_budget=BUDGET)
    per_gate = max(1e-4, (time.perf_counter() - t0) / 4)
    m = int(max(8, min(len(rzz), budget_s * 0.6 / per_gate - len(rx))))
    stride = max(1, len(rzz) // m)
    sub = R.CircuitIR(num_qubits=n_run, gates=hs + rzz[::stride] + rx)
    _, rec = R.run_circuit_sharded(sub, plan, precision, memory_budget=BUDGET)
    rows = rec.gates
    t_rzz = [r.compute_s + r.exchange_s for r in rows if r.kind == "RZZ"]
    t_rx = [r.compute_s + r.exchange_s for r in rows if r.kind == "RX"]
    # the coordinator's per-gate barrier and queue traffic are part of the
    # reference's cost: spread the wall time not in the rows over the gates
    overhead = max(0.0, rec.wall_seconds - sum(r.compute_s + r.exchange_s for r in rows)) / len(rows)
    t_layer = (E * (statistics.mean(t_rzz) + overhead) + n * (statistics.mean(t_rx) + overhead)) * scale
    # single thread: the dense engine on a prefix of the same gates
    n1 = min(n_run, 26)
    inst1 = R.generate_instance(n1, seed)
    c1 = R.build_circuit(inst1, R.LrQaoaParams(p=p))
    E1 = n1 * (n1 - 1) // 2
    g1 = c1.gates[n1:n1 + E1 + n1]
    r1 = [g for g in g1 if g.kind == "RZZ"]
    x1 = [g for g in g1 if g.kind == "RX"]
    budget1 = budget_s * 0.35
    sv = R.zero_state(n1, precision, memory_budget=BUDGET)
    from lrqbench.engine import _apply_gate_kernel  # the reference's own per-gate kernels

    ts_r, ts_x = [], []
    t0 = time.perf_counter()
    k = 0
    while (time.perf_counter() - t0 < budget1 or len(ts_x) < 2) and k < len(r1):
        g = r1[(k * 37) % len(r1)]
        s = time.perf_counter()
        _apply_gate_kernel(sv.amps, g, g.qubits)
        ts_r.append(time.perf_counter() - s)
        if k % 8 == 0:
            g = x1[k % len(x1)]
            s = time.perf_counter()
            _apply_gate_kernel(sv.amps, g, g.qubits)
            ts_x.append(time.perf_counter() - s)
        k += 1
    del sv
    t_layer1 = (E * statistics.mean(ts_r) + n * statistics.mean(ts_x)) * float(1 << (n - n1))
    return {"value": (1 << n) / t_layer, "unit": "amp-updates/s", "cores": G, "kind": "reference",
            "sample": (f"lrqbench (baseline/_ref) run_circuit_sharded, {G} shard threads, at n={n_run}: "
                       f"{len(hs)} H + {len(t_rzz)} RZZ (every {stride}th of layer 0) + {len(t_rx)} RX gates, "
                       f"mean per-gate time incl. exchange and barrier x (E_n RZZ + n RX) per layer, "
                       f"x{int(scale)} to n={n} (per-gate cost is linear in 2^n)"),
            "t_layer_s": t_layer,
            "single_thread": {"value": (1 << n) / t_layer1, "unit": "amp-updates/s", "cores": 1,
                              "sample": f"lrqbench run_circuit's per-gate kernels (engine.py:158-166) at n={n1}: "
                                        f"{len(ts_r)} RZZ + {len(ts_x)} RX, x{1 << (n - n1)} to n={n}",
                              "t_layer_s": t_layer1}}


# ---------------------------------------------------------------------------


def device_run(dev, lay, u, steps, warmup, clock_index=None):
    """Time `steps` runs + samples on the engine stream (CUDA events)."""
    import torch

    stream = torch.cuda.ExternalStream(dev.stream())
    # the warm-up runs' fused final pass also searches the max cut (C*, the
    # denominator of r); the timed runs know it and only sum p and p*C, as
    # run_circuit does for a solved instance
    dev.set_search(True)
    for _ in range(warmup):
        dev.run(lay.phase, lay.mixer)
        dev.sample(u)
    red0 = dev.reduce()
    dev.set_search(False)
    dev.set_timing(True)
    ms_all, kinds_all = [], ""
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(clock_index) if clock_index is not None else None
    if clk:
        clk.__enter__()
    try:
        e0.record(stream)
        for _ in range(steps):
            dev.run(lay.phase, lay.mixer)
            ms, kinds = dev.timings()
            ms_all += ms
            kinds_all += kinds
            dev.sample(u)
        e1.record(stream)
        e1.synchronize()
    finally:
        if clk:
            clk.__exit__(None, None, None)
    torch.cuda.synchronize()
    dev.set_timing(False)
    dev.search_result = red0
    return e0.elapsed_time(e1), ms_all, kinds_all, (clk.summary() if clk else None)


def extra_config(L, _native, cfg, steps, peak):
    """A BASELINE config measured on the device (no e2e, no CPU arm)."""
    n, p, prec, shots = CONFIGS[cfg]
    n = min(n, 33)
    B = 8 if prec == "fp32" else 16
    inst = L.generate_instance(n, 1)
    lay = L.lower_circuit(L.build_circuit(inst, L.LrQaoaParams(p=p)))
    u = L.derive_rng(1, "shots", 0).random(shots)
    dev = _native.DeviceState(n, B)
    dev.set_cost(inst.weights())
    dev_ms, ms, kinds, _ = device_run(dev, lay, u, steps, 2)
    red = dev.search_result
    dev.close(park=False)
    _native.drain_pool()
    pk = per_kernel(ms, kinds, sweep_labels(n, B, p, 1), n, B, peak, steps)
    dk, dv = dominant(pk, peak)
    return {"workload": f"BASELINE configs[{cfg - 1}]: n={n} p={p} {'complex64' if B == 8 else 'complex128'}",
            "value": float(1 << n) * p * steps / (dev_ms * 1e-3), "ms_per_step": dev_ms / steps,
            "ms_per_layer": dev_ms / steps / p, "dominant_kernel": {dk: dv}, "per_kernel": pk,
            "sum_p": red.sum_p, "max_cut_E": red.min_energy}


def sample_check(L, circ, solved, prec, shots=10000, groups=40):
    """Untimed: chi-square of `shots` samples of the run's state against the
    exact distribution of C (the device histogram pass), grouped into ~40
    equiprobable bins (north_star: sampled histograms must pass chi-square)."""
    from scipy import stats

    sv = L.run_circuit(circ, prec, memory_budget=BUDGET)
    try:
        d = L.exact_cut_distribution(sv, solved, bins=2048)
        shot_set = L.sample(sv, shots, 3)
    finally:
        sv.release()
    p = d.probs / d.probs.sum()
    gid = np.minimum((np.cumsum(p) * groups).astype(int), groups - 1)
    exp_g = np.bincount(gid, weights=p, minlength=groups) * shots
    obs_g = np.bincount(gid[d.bin_of(L.cut_values(solved, shot_set.indices))], minlength=groups).astype(float)
    keep = exp_g > 5
    chi2 = float(np.sum((obs_g[keep] - exp_g[keep]) ** 2 / exp_g[keep]))
    df = int(keep.sum()) - 1
    other_o, other_e = obs_g[~keep].sum(), exp_g[~keep].sum()
    if other_e > 5:
        chi2 += (other_o - other_e) ** 2 / other_e
        df += 1
    return {"shots": shots, "bins": int(df + 1), "chi2": chi2, "df": df, "p_value": float(stats.chi2.sf(chi2, df)),
            "source": "exact C histogram from the device pass (lrq_set_histogram), 2048 fine bins grouped ~equiprobable"}


def run_ours(args, rank, world, local_rank, dist):
    os.environ.setdefault("LRQ_DEVICE", str(local_rank))
    import paper_2604_26423_b200 as L
    from paper_2604_26423_b200 import _native
    from paper_2604_26423_b200.build import build

    if rank == 0:
        build()
    barrier(dist)
    import torch

    dev_index = int(os.environ["LRQ_DEVICE"])
    torch.cuda.set_device(dev_index)
    n, p, prec, shots, label, scaling = workload(args, world)
    B = 8 if prec == "fp32" else 16
    inst = L.generate_instance(n, args.seed)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=p))
    lay = L.lower_circuit(circ)
    w = inst.weights()
    u = L.derive_rng(1, "shots", 0).random(shots)
    peak, peak_kind = measured_peak()

    # --- device-resident measurement (value) --------------------------------
    dev = _native.DeviceState(n, B)
    dev.set_cost(w)
    barrier(dist)
    dev_ms, ms_all, kinds_all, clocks = device_run(dev, lay, u, args.steps, max(1, args.warmup), dev_index)
    barrier(dist)
    dev_ms_max = max_over_ranks(dist, dev_ms)
    red = dev.reduce()
    srch = dev.search_result
    dev.close(park=False)
    _native.drain_pool()

    # --- end to end through the public API (e2e) ------------------------------
    z = int(srch.argmax_cut)
    solved = L.WmcInstance(inst.num_vertices, inst.edges, inst.seed,
                           L.OptimalCut(L.index_to_bitstring(z, n), float(L.cut_values(inst, [z])[0])))
    # the drop-in API as a user calls it: the circuit of the solved instance
    # (C* known: the final pass skips the max-cut search, as in the device
    # loop), an explicit budget, and a dropped StateVector's HBM parked for
    # the next run_circuit of the same shape (no cudaMalloc per step)
    circ = L.build_circuit(solved, L.LrQaoaParams(p=p))
    sv = L.run_circuit(circ, prec, memory_budget=BUDGET)
    L.exact_expected_r(sv, solved)
    L.sample(sv, shots, 1)
    del sv
    barrier(dist)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sv = L.run_circuit(circ, prec, memory_budget=BUDGET)
        r_exact = L.exact_expected_r(sv, solved)
        shots_set = L.sample(sv, shots, 1)
        del sv
    e2e_s_max = max_over_ranks(dist, time.perf_counter() - t0)
    r_sampled = L.approximation_ratio(solved, shots_set)
    chi = sample_check(L, circ, solved, prec)  # untimed: 10k shots against the exact C distribution
    _native.drain_pool()

    extra = {}
    if world == 1 and not args.no_extra_configs and not args.n:
        for cfg in (2, 4):
            try:
                extra[f"configs[{cfg - 1}]"] = extra_config(L, _native, cfg, 3, peak)
            except Exception as exc:  # noqa: BLE001 - reported, not fatal
                extra[f"configs[{cfg - 1}]"] = {"error": str(exc)[:200]}
    if rank != 0:
        return None
    labels = sweep_labels(n, B, p, 1)
    pk = per_kernel(ms_all, kinds_all, labels, n, B, peak, args.steps)
    dk, dv = dominant(pk, peak)
    traffic = profiled_traffic().get(f"n{n}_{prec}", {})
    traffic = traffic if isinstance(traffic, dict) else {}
    tr = [traffic[lab] for lab in dv["labels"] if lab in traffic]
    launches_per_step = kernel_launches(kinds_all, n) // args.steps + 1  # + sample kernel
    amp_updates = float(1 << n) * p * args.steps * world
    E = n * (n - 1) // 2
    h2d = lay.phase.nbytes + lay.mixer.nbytes + w.nbytes + shots * 8
    d2h = shots * 8 + 40
    cpu = cpu_reference(n, p, prec, args.cpu_seconds, args.seed) if world == 1 else None
    return {
        "metric": METRIC,
        "value": amp_updates / (dev_ms_max * 1e-3),
        "unit": "amp-updates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dev_ms_max / args.steps,
        "ms_per_layer": dev_ms_max / args.steps / p,
        "gate_equiv_amp_updates_per_s": amp_updates * (E + n) / (dev_ms_max * 1e-3),
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "c64 (fp32 amplitudes, fp64 phases and reductions)" if B == 8 else "c128 (fp64)",
        "data": "synthetic: generate_instance(n, seed) Philox weights, LrQaoaParams(p) default ramp",
        "config": {"workload": label, "n": n, "p": p, "precision": prec, "shots": shots,
                   "state_bytes": B << n, "parallelism": f"replicas x{world}",
                   "l2": f"state ({(B << n) >> 30} GiB) >> L2 (126 MB); no flush needed"},
        "e2e": {"value": amp_updates / e2e_s_max, "unit": "amp-updates/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "api": "run_circuit -> exact_expected_r -> sample (drop-in API, ctypes C-ABI)"},
        "roofline": {"bound": "hbm", "kernel": f"{dk} ({', '.join(dv['labels'])})", "achieved": dv["achieved"],
                     "peak": peak, "unit": "GB/s", "frac": dv["frac"], "peak_source": peak_kind,
                     "traffic": (sum(tr) / len(tr)) if tr else None,
                     "bytes_per_launch": dv["bytes_per_launch_avg"], "launch_ms_avg": dv["launch_ms_avg"],
                     "time_share": dv["time_share"], "per_kernel": pk},
        "sweeps_per_step": sum(v["launches_per_step"] for v in pk.values()),
        "gpu_launches": launches_per_step * args.steps,
        "cpu_baseline": None if cpu is None else {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                                      "single_thread")},
        "clocks": clocks,
        "configs": extra,
        "results": {"exact_r": r_exact, "sampled_r": r_sampled, "sum_p": red.sum_p,
                    "max_cut": solved.optimal_cut.value,
                    "min_cut": 0.5 * (inst.total_weight() - srch.max_energy),
                    "chi_square": chi},
    }


def run_ours_dist(args, rank, world, local_rank, dist):
    """N > 1: one distributed state (default: 2^33 complex128 amplitudes per GPU)."""
    os.environ.setdefault("LRQ_DEVICE", str(local_rank))
    import paper_2604_26423_b200 as L
    from paper_2604_26423_b200 import _native
    from paper_2604_26423_b200.build import build
    from paper_2604_26423_b200.distributed import drain_dist_pool, enable_peer_remap, run_circuit_distributed

    if rank == 0:
        build()
    barrier(dist)
    import torch

    dev_index = int(os.environ["LRQ_DEVICE"])
    torch.cuda.set_device(dev_index)
    g = world.bit_length() - 1
    if (1 << g) != world:
        raise SystemExit("--gpus must be a power of two")
    n, p, prec, shots, label, scaling = workload(args, world)
    nl = n - g
    B = 8 if prec == "fp32" else 16
    inst = L.generate_instance(n, args.seed)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=p))
    lay = L.lower_circuit(circ)
    w = inst.weights()
    u = L.derive_rng(1, "shots", 0).random(shots)
    peak, peak_kind = measured_peak()

    box = [_native.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    dev = _native.DeviceState.create_dist(n, B, dev_index, rank, world, box[0])
    mode = enable_peer_remap(dev)
    dev.set_cost(w)
    barrier(dist)
    dev_ms, ms_all, kinds_all, clocks = device_run(dev, lay, u, args.steps, max(1, args.warmup), dev_index)
    barrier(dist)
    dev_ms_max = max_over_ranks(dist, dev_ms)
    red = dev.reduce()
    srch = dev.search_result
    dev.close()

    z = int(srch.argmax_cut)
    solved = L.WmcInstance(inst.num_vertices, inst.edges, inst.seed,
                           L.OptimalCut(L.index_to_bitstring(z, n), float(L.cut_values(inst, [z])[0])))
    circ = L.build_circuit(solved, L.LrQaoaParams(p=p))
    sv = run_circuit_distributed(circ, prec, memory_budget=BUDGET)  # warm: communicator, pooled shard
    sv.exact_expected_r(solved)
    sv.sample(shots, 1)
    sv.release()
    barrier(dist)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sv = run_circuit_distributed(circ, prec, memory_budget=BUDGET)
        r_exact = sv.exact_expected_r(solved)
        shots_set = sv.sample(shots, 1)
        sv.release()
    e2e_s_max = max_over_ranks(dist, time.perf_counter() - t0)
    r_sampled = L.approximation_ratio(solved, shots_set)
    drain_dist_pool()
    _native.drain_pool()
    if rank != 0:
        return None

    labels = sweep_labels(nl, B, p, world)
    pk = per_kernel(ms_all, kinds_all, labels, nl, B, peak, args.steps)
    dk, dv = dominant(pk, peak)
    # remap timing: 'Y' fused (the carrying sweep + barrier), 'W' pipelined
    # (the block-split sweep with the swaps overlapped + the exposed tail),
    # 'T' serial exchange
    remap_ms, exposed = [], []
    for i, k in enumerate(kinds_all):
        if k == "T":
            remap_ms.append(ms_all[i])
            exposed.append(ms_all[i])
        elif k in "YW":
            remap_ms.append(ms_all[i] + (ms_all[i - 1] if i > 0 else 0.0))
            exposed.append(ms_all[i])
    sent = (world - 1) * (B << (nl - g))  # bytes sent (= received) per GPU per remap
    algbw = sent / (statistics.mean(remap_ms) * 1e-3) / 1e9 if remap_ms else None
    amp_updates = float(1 << n) * p * args.steps
    E = n * (n - 1) // 2
    swaps_per_remap = world - 1 if mode != "fused" else 0
    launches_per_step = (kernel_launches(kinds_all, nl) + swaps_per_remap * sum(k in "WT" for k in kinds_all)) \
        // args.steps + 1
    return {
        "metric": METRIC,
        "value": amp_updates / (dev_ms_max * 1e-3),
        "unit": "amp-updates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dev_ms_max / args.steps,
        "ms_per_layer": dev_ms_max / args.steps / p,
        "gate_equiv_amp_updates_per_s": amp_updates * (E + n) / (dev_ms_max * 1e-3),
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "c64 (fp32 amplitudes, fp64 phases and reductions)" if B == 8 else "c128 (fp64)",
        "data": "synthetic: generate_instance(n, seed) Philox weights, LrQaoaParams(p) default ramp",
        "config": {"workload": label, "n": n, "n_local": nl, "p": p, "precision": prec, "shots": shots,
                   "state_bytes": B << n, "parallelism": f"global-qubit sharding x{world}, one remap per layer ({mode})",
                   "l2": "shard >> L2 (126 MB); no flush needed"},
        "e2e": {"value": amp_updates / e2e_s_max, "unit": "amp-updates/s",
                "h2d_bytes_per_step": int(lay.phase.nbytes + lay.mixer.nbytes + w.nbytes + shots * 8),
                "d2h_bytes_per_step": int(shots * 8 + 40 * world),
                "api": "run_circuit_distributed -> exact_expected_r -> sample (collective, ctypes C-ABI)"},
        "roofline": {"bound": "hbm", "kernel": f"{dk} ({', '.join(dv['labels'])}; local shard)",
                     "achieved": dv["achieved"], "peak": peak, "unit": "GB/s", "frac": dv["frac"],
                     "peak_source": peak_kind, "traffic": None, "bytes_per_launch": dv["bytes_per_launch_avg"],
                     "launch_ms_avg": dv["launch_ms_avg"], "time_share": dv["time_share"], "per_kernel": pk},
        "remap": {"mode": mode, "per_step": len(remap_ms) // args.steps,
                  "ms_avg": statistics.mean(remap_ms) if remap_ms else None,
                  "exposed_ms_avg": statistics.mean(exposed) if exposed else None,
                  "ms_note": "fused/pipelined: the carrying group-A sweep plus the barrier / exposed tail; serial: the exchange",
                  "bytes_sent_per_gpu": sent, "algbw_GBps": algbw,
                  "busbw_GBps": algbw * (world - 1) / world if algbw else None, "nvlink_peak_GBps_per_dir": 900},
        "gpu_launches": launches_per_step * args.steps,
        "cpu_baseline": None,
        "clocks": clocks,
        "results": {"exact_r": r_exact, "sampled_r": r_sampled, "sum_p": red.sum_p,
                    "max_cut": solved.optimal_cut.value},
    }


def run_reference(args, rank, world):
    if rank != 0:
        return None
    n, p, prec, shots, label, scaling = workload(args, world)
    cpu = cpu_reference(n, p, prec, args.cpu_seconds, args.seed)
    t_step = cpu["t_layer_s"] * p
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": cpu["value"],
        "unit": "amp-updates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_step * 1e3,
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "c64" if prec == "fp32" else "c128",
        "data": "synthetic",
        "config": {"workload": label + " - the reference's CPU engine on the host cores", "n": n, "p": p,
                   "precision": prec, "shots": shots},
        "cpu_baseline": {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample", "single_thread")},
        "e2e": {"value": cpu["value"], "unit": "amp-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        dist = init_dist(world)
        try:
            out = (run_ours_dist if world > 1 else run_ours)(args, rank, world, local_rank, dist)
        except Exception as exc:  # one parsable line saying what failed, then a failing exit
            if rank == 0:
                print(json.dumps({"metric": METRIC, "value": None, "n_gpus": world, "error": f"{type(exc).__name__}: {exc}"}),
                      flush=True)
            raise
        if dist is not None:
            dist.destroy_process_group()
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
