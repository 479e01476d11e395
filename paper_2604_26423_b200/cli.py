"""Command line for the GPU path: ``gen`` and ``simulate`` (noiseless and noisy).

This is the ``lrqbench simulate`` integration of SURVEY §8(f) rank 1
(cli.py:156-244 of the reference): the same arguments, results JSON keys,
``<out>.timing.csv`` for sharded runs and ``<out>.manifest.json``, with the
circuit run by liblrq.so; ``--mode noisy`` runs the GPU trajectories
(noise.py).  ``classify``, ``bench``, ``fitnoise``, ``hqc`` and ``replay``
are off the hot path.

    python -m paper_2604_26423_b200 gen --n 26 --out inst.json --solve-limit 26
    python -m paper_2604_26423_b200 simulate --instance inst.json --out res.json --p 3 --precision fp64

Exit codes (cli.py:64-67): 0 success, 2 bad input, 3 over a capacity
limit, 4 runtime failure.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
from datetime import datetime, timezone
from pathlib import Path

from . import __version__
from .circuit import LrQaoaParams, build_circuit, gate_counts
from .engine import exact_expected_r, run_circuit, sample, save_statevector
from .noise import DepolarizingConfig, epsilon_accumulated, r_overlap, run_noisy_ensemble
from .errors import AbortedRunError, CapacityError, StateError, ValidationError
from .problem import (approximation_ratio, generate_instance, load_instance, random_baseline_expectation,
                      save_instance, solve_instance)
from .rng import derive_seed
from .sharded import plan_for_shard_count, run_circuit_sharded, write_timing_csv

EXIT_OK, EXIT_VALIDATION, EXIT_CAPACITY, EXIT_RUNTIME = 0, 2, 3, 4


def _sha256(path: Path) -> str:
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        for chunk in iter(lambda: fh.read(1 << 20), b""):
            h.update(chunk)
    return h.hexdigest()


def _manifest(args, inputs: list[Path], outputs: list[Path]) -> Path:
    params = {k: (str(v) if isinstance(v, Path) else v) for k, v in vars(args).items()
              if k not in ("func", "argv") and not callable(v)}
    doc = {
        "tool": "paper_2604_26423_b200",
        "version": __version__,
        "backend": "cuda",
        "command": args.command,
        "argv": list(args.argv),
        "params": params,
        "timestamp_utc": datetime.now(timezone.utc).isoformat(),
        "inputs": {str(p): _sha256(Path(p)) for p in inputs},
        "outputs": {str(p): _sha256(Path(p)) for p in outputs},
    }
    path = Path(str(outputs[0]) + ".manifest.json")
    path.write_text(json.dumps(doc, indent=2, sort_keys=True) + "\n")
    return path


def _cmd_gen(args) -> int:
    inst = generate_instance(args.n, args.seed)
    if args.n <= args.solve_limit:
        inst = solve_instance(inst, limit=args.solve_limit)
    else:
        print(f"warning: n={args.n} exceeds solve limit {args.solve_limit}; optimal cut omitted", file=sys.stderr)
    save_instance(inst, args.out)
    _manifest(args, [], [args.out])
    opt = "null" if inst.optimal_cut is None else f"{inst.optimal_cut.value:.6f}"
    print(f"wrote {args.out}: n={args.n} edges={inst.num_edges} optimal={opt}")
    return EXIT_OK


def _cmd_simulate(args) -> int:
    inst = load_instance(args.instance)
    db = args.delta if args.delta_beta is None else args.delta_beta
    dg = args.delta if args.delta_gamma is None else args.delta_gamma
    circuit = build_circuit(inst, LrQaoaParams(p=args.p, delta_beta=db, delta_gamma=dg))
    n_1q, n_2q = gate_counts(inst.num_vertices, args.p)
    solved = inst.optimal_cut is not None
    payload = {"n": inst.num_vertices, "p": args.p, "delta_beta": db, "delta_gamma": dg, "seed": args.seed,
               "precision": args.precision, "n_1q": n_1q, "n_2q": n_2q, "mode": args.mode}
    outputs = [args.out]
    if args.mode == "noisy":
        return _simulate_noisy(args, inst, circuit, n_2q, solved, payload, outputs)
    if args.shards > 1:
        plan = plan_for_shard_count(inst.num_vertices, args.shards)
        sv, record = run_circuit_sharded(circuit, plan, args.precision, args.memory_bytes)
        timing = args.out.with_suffix(".timing.csv")
        with open(timing, "w", newline="") as fh:
            write_timing_csv([record], fh)
        outputs.append(timing)
    else:
        sv = run_circuit(circuit, args.precision, args.memory_bytes)
    shots = sample(sv, args.shots, args.seed)
    payload.update({
        "shards": args.shards,
        "shots": args.shots,
        "mean_r": approximation_ratio(inst, shots) if solved else None,
        "exact_expected_r": exact_expected_r(sv, inst) if solved else None,
        "bitstrings": shots.bitstrings(),
    })
    if args.dump_state is not None:
        save_statevector(sv, args.dump_state)
        outputs.append(args.dump_state)
    sv.release()
    args.out.write_text(json.dumps(payload, indent=2, sort_keys=True) + "\n")
    _manifest(args, [args.instance], outputs)
    shown = "n/a" if payload["mean_r"] is None else f"{payload['mean_r']:.4f}"
    print(f"wrote {args.out}: mode={args.mode} mean_r={shown}")
    return EXIT_OK


def _simulate_noisy(args, inst, circuit, n_2q, solved, payload, outputs) -> int:
    """cli.py:195-232 of the reference: pooled trajectory shots, and against
    the ideal and random baselines the overlap ratio."""
    cfg = DepolarizingConfig(epsilon=args.epsilon, trajectories=args.trajectories, rng_seed=args.seed)
    shots = run_noisy_ensemble(circuit, cfg, args.shots, args.precision, args.memory_bytes)
    mean_r = approximation_ratio(inst, shots) if solved else None
    ovl = None
    if solved:
        ideal = run_circuit(circuit, args.precision, args.memory_bytes)
        if args.ideal_shots is None:
            r_ideal = exact_expected_r(ideal, inst)
        else:
            r_ideal = approximation_ratio(inst, sample(ideal, args.ideal_shots, derive_seed(args.seed, "ideal")))
        ideal.release()
        r_random = random_baseline_expectation(inst)
        ovl = r_overlap(mean_r, r_random, r_ideal)
        payload.update({"r_ideal": r_ideal, "r_random": r_random})
    payload.update({"epsilon": args.epsilon, "trajectories": args.trajectories, "shots": args.shots,
                    "eps_acc": epsilon_accumulated(n_2q, args.epsilon), "mean_r": mean_r, "r_ovl": ovl,
                    "bitstrings": shots.bitstrings()})
    args.out.write_text(json.dumps(payload, indent=2, sort_keys=True) + "\n")
    _manifest(args, [args.instance], outputs)
    shown = "n/a" if payload["mean_r"] is None else f"{payload['mean_r']:.4f}"
    print(f"wrote {args.out}: mode={args.mode} mean_r={shown}")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2604_26423_b200",
                                 description="LR-QAOA MaxCut simulation on B200 (lrqbench-compatible gen/simulate)")
    ap.add_argument("--version", action="version", version=f"%(prog)s {__version__}")
    sub = ap.add_subparsers(dest="command", required=True)

    def common(p):
        p.add_argument("--seed", type=int, default=0, help="seed for every derived stream")
        p.add_argument("--threads", type=int, default=int(os.environ.get("LRQBENCH_THREADS", "1") or 1),
                       help="accepted for compatibility; the GPU path does not use host threads")

    g = sub.add_parser("gen", help="generate a weighted MaxCut instance")
    g.add_argument("--n", type=int, required=True)
    g.add_argument("--out", type=Path, required=True)
    g.add_argument("--solve-limit", type=int, default=24)
    common(g)
    g.set_defaults(func=_cmd_gen)

    s = sub.add_parser("simulate", help="run the circuit for an instance")
    s.add_argument("--instance", type=Path, required=True)
    s.add_argument("--out", type=Path, required=True, help="results JSON path")
    s.add_argument("--p", type=int, default=3)
    s.add_argument("--delta", type=float, default=0.2)
    s.add_argument("--delta-beta", type=float, default=None)
    s.add_argument("--delta-gamma", type=float, default=None)
    s.add_argument("--mode", choices=("noiseless", "noisy"), default="noiseless")
    s.add_argument("--shots", type=int, default=100)
    s.add_argument("--shards", type=int, default=1)
    s.add_argument("--precision", choices=("fp32", "fp64"), default="fp32")
    s.add_argument("--epsilon", type=float, default=0.0, help="two-qubit depolarizing rate")
    s.add_argument("--trajectories", type=int, default=1)
    s.add_argument("--ideal-shots", type=int, default=None,
                   help="estimate the ideal baseline from this many shots instead of exactly")
    s.add_argument("--dump-state", type=Path, default=None)
    s.add_argument("--memory-bytes", type=int, default=None)
    common(s)
    s.set_defaults(func=_cmd_simulate)
    return ap


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    args.argv = list(sys.argv[1:] if argv is None else argv)
    try:
        return args.func(args)
    except ValidationError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_VALIDATION
    except CapacityError as exc:
        print(f"capacity error: {exc}", file=sys.stderr)
        return EXIT_CAPACITY
    except (StateError, AbortedRunError, OSError) as exc:
        print(f"runtime error: {exc}", file=sys.stderr)
        return EXIT_RUNTIME


if __name__ == "__main__":
    sys.exit(main())
