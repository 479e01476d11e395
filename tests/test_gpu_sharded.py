"""GPU tests of the sharded engine: G shard states of an in-process shard
group on one device, running the distributed sweep plan (per-layer remaps,
rank-local phase terms, final reduction in the identity permutation,
rank-partitioned sampler).  This exercises every part of the multi-GPU
engine except the NCCL calls themselves.

Tolerances as in test_gpu_parity: amplitudes normwise 1e-10 (complex128) /
1e-5 (complex64) against the oracle; sharded vs dense 1e-12 (complex128).
"""
import numpy as np
import pytest

import paper_2604_26423_b200 as L
from oracle import lrq_oracle as O
from paper_2604_26423_b200 import _native

pytestmark = pytest.mark.gpu

TOL = {"fp64": 1e-10, "fp32": 1e-5}


def normwise(got, want):
    return float(np.linalg.norm(got.astype(np.complex128) - want) / np.linalg.norm(want))


@pytest.fixture(scope="module", autouse=True)
def _engine():
    from paper_2604_26423_b200.build import build
    build()
    assert _native.device_count() >= 1, "GPU tests need a CUDA device"


@pytest.mark.parametrize("n,G,p,prec,dbeta", [
    (16, 2, 3, "fp64", 0.2),   # odd p: restoring remap
    (16, 2, 2, "fp64", 1.2),   # one deferred-X layer: mirror exchange at the end
    (17, 4, 3, "fp64", 1.2),   # flips + odd p
    (18, 8, 2, "fp64", 0.2),
    (18, 4, 4, "fp32", 0.2),
    (19, 2, 5, "fp32", 1.0),
    # short last group: the top local qubits come from the group below
    (17, 8, 3, "fp64", 0.9),
    (17, 8, 3, "fp64", 0.2),
    (15, 4, 2, "fp64", 0.2),
    (17, 8, 2, "fp32", 0.2),
])
def test_sharded_matches_oracle_and_dense(n, G, p, prec, dbeta):
    inst = L.solve_instance(L.generate_instance(n, 3))
    circ = L.build_circuit(inst, L.LrQaoaParams(p=p, delta_beta=dbeta))
    plan = L.plan_for_shard_count(n, G)
    sv, rec = L.run_circuit_sharded(circ, plan, prec)
    try:
        assert isinstance(sv, L.ShardedStateVector)
        assert rec.num_shards == G and rec.nq == n
        assert rec.amps_exchanged == L.remap_volume(circ, plan, prec)
        assert rec.compute_seconds > 0 and rec.exchange_seconds > 0
        got = sv.amps
        assert got.dtype == (np.complex128 if prec == "fp64" else np.complex64)
        want = O.simulate(n, inst.weights(), p, "fp64", dbeta=dbeta)
        assert normwise(got, want) < TOL[prec]
        dense = L.run_circuit(circ, prec)
        if prec == "fp64":
            assert normwise(got, dense.amps.astype(np.complex128)) < 1e-12
        r_sh = L.exact_expected_r(sv, inst)
        r_de = L.exact_expected_r(dense, inst)
        assert r_sh == pytest.approx(r_de, rel=1e-12 if prec == "fp64" else 1e-6)
        assert sv.norm_squared() == pytest.approx(1.0, rel=TOL[prec])
        s_sh = L.sample(sv, 3000, rng_seed=1).indices
        s_de = L.sample(dense, 3000, rng_seed=1).indices
        assert int(np.sum(s_sh != s_de)) <= 2
        # a cost the run was not fused with: recompute on every shard
        other = L.solve_instance(L.generate_instance(n, 9))
        assert L.exact_expected_r(sv, other) == pytest.approx(L.exact_expected_r(dense, other),
                                                               rel=1e-12 if prec == "fp64" else 1e-6)
        dense.release()
    finally:
        sv.release()


def test_small_shards_run_dense_bitwise():
    inst = L.generate_instance(8, 31)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=3))
    dense = L.run_circuit(circ, "fp64").amps.copy()
    for G in (1, 2, 4, 8):
        sv, rec = L.run_circuit_sharded(circ, L.plan_for_shard_count(8, G), "fp64")
        np.testing.assert_array_equal(sv.amps, dense)
        assert rec.num_shards == G and rec.amps_exchanged == 0
        sv.release()


def test_sharded_state_copy_range_and_dump(tmp_path):
    inst = L.generate_instance(16, 2)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=2))
    sv, _ = L.run_circuit_sharded(circ, L.plan_for_shard_count(16, 4), "fp64")
    try:
        full = sv.amps
        np.testing.assert_array_equal(sv._copy_range(1000, 40000), full[1000:41000])
        np.testing.assert_array_equal(sv.shard_amps(3), full[3 << 14:])
        path = tmp_path / "s.lqsv"
        L.save_statevector(sv, path)
        from paper_2604_26423_b200.engine import load_statevector_amps
        n, back = load_statevector_amps(path)
        assert n == 16
        np.testing.assert_array_equal(back, full)
    finally:
        sv.release()


def test_worker_failure_aborts_run(monkeypatch):
    circ = L.build_circuit(L.generate_instance(16, 0), L.LrQaoaParams(p=2))
    real = _native.DeviceState.run
    calls = {"n": 0}

    def flaky(self, phase, mixer):
        calls["n"] += 1
        if calls["n"] == 2:
            raise RuntimeError("injected shard fault")
        return real(self, phase, mixer)

    monkeypatch.setattr(_native.DeviceState, "run", flaky)
    with pytest.raises(L.AbortedRunError):
        L.run_circuit_sharded(circ, L.plan_for_shard_count(16, 4), "fp64")


def test_scaling_sweeps():
    recs = L.scaling_sweep(L.SweepConfig(mode="strong", nq=16, shard_counts=(1, 2, 4), p=1, precision="fp64"))
    assert [r.num_shards for r in recs] == [1, 2, 4]
    vols = [r.amps_exchanged for r in recs]
    assert vols[0] == 0 and 0 < vols[1] < vols[2]
    recs = L.scaling_sweep(L.SweepConfig(mode="size", nq_values=(16, 17, 18), nq_local=15, p=2, precision="fp64"))
    vols = [r.amps_exchanged for r in recs]
    assert vols == sorted(vols) and vols[0] < vols[-1]


@pytest.mark.parametrize("n,G,p,prec,dbeta", [(26, 2, 3, "fp32", 1.2), (24, 4, 2, "fp64", 0.2), (26, 8, 3, "fp64", 0.9)])
def test_larger_sharded_runs_match_dense(n, G, p, prec, dbeta):
    """Three-group local plans: the shards' P/F sweeps on Z run the
    warp-decoupled kernel with rank-local fields; checked against the dense
    engine (itself checked against the oracle)."""
    inst = L.generate_instance(n, 4)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=p, delta_beta=dbeta))
    sv, rec = L.run_circuit_sharded(circ, L.plan_for_shard_count(n, G), prec)
    try:
        assert isinstance(sv, L.ShardedStateVector)
        dense = L.run_circuit(circ, prec)
        tol = 1e-12 if prec == "fp64" else 3e-6
        assert normwise(sv.amps, dense.amps.astype(np.complex128)) < tol
        dense.release()
    finally:
        sv.release()


REMAP_MODES = {"fused": ("1", "1", "Y"), "pipelined": ("0", "1", "W"), "serial": ("0", "0", "T")}


@pytest.mark.parametrize("n,G,p,prec", [(16, 2, 3, "fp64"), (18, 4, 2, "fp32"), (26, 8, 3, "fp64"),
                                        (27, 8, 4, "fp32"), (25, 2, 3, "fp64")])
def test_remap_transports_are_bitwise_equal(monkeypatch, n, G, p, prec):
    """The three remap forms move exactly the same amplitudes, so the states
    are bitwise identical: fused (the group-A sweep stores each block into
    its owner's spare buffer), pipelined (the group-A sweep runs block by
    block in XOR order and each finished block is swapped in place with its
    owner on a second stream while the next block is swept: the form used
    when no spare buffer fits) and serial (sweep, then the XOR swaps)."""
    circ = L.build_circuit(L.generate_instance(n, 6), L.LrQaoaParams(p=p, delta_beta=0.9))
    out = {}
    for mode, (fused, pipe, tag) in REMAP_MODES.items():
        monkeypatch.setenv("LRQ_FUSED_REMAP", fused)
        monkeypatch.setenv("LRQ_PIPELINED_REMAP", pipe)
        sv, rec = L.run_circuit_sharded(circ, L.plan_for_shard_count(n, G), prec)
        kinds = [g.kind for g in rec.gates]
        out[mode] = (sv.amps.copy(), kinds, L.sample(sv, 500, rng_seed=2).indices)
        assert tag in kinds, (mode, kinds)
        sv.release()
    for mode in ("pipelined", "serial"):
        np.testing.assert_array_equal(out[mode][0], out["fused"][0])
        np.testing.assert_array_equal(out[mode][2], out["fused"][2])
    # the same sweeps; only the remap records differ (the odd-p restoring
    # remap follows a high-group sweep and is never fused or pipelined)
    strip = lambda ks: [k for k in ks if k not in "YWT"]  # noqa: E731
    assert strip(out["fused"][1]) == strip(out["pipelined"][1]) == strip(out["serial"][1])


def test_shards_at_the_hbm_limit_take_the_pipelined_remap():
    """n=33 complex128 over 8 shards on ONE B200: 8 x 16 GiB = 128 GiB, so
    the fused remap's spare buffers (another 128 GiB) do not fit and the
    group takes the in-place pipelined remap.  Checked against the dense
    complex128 run of the same circuit (run first, then freed): exact r,
    norm, the max-cut argmax, sampled shots and amplitude ranges."""
    n, G, p = 33, 8, 3
    inst = L.generate_instance(n, 1)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=p))
    budget = 1 << 40
    dense = L.run_circuit(circ, "fp64", memory_budget=budget)
    red_d = dense.device_state.reduce()
    rng = np.random.default_rng(0)
    starts = [int(x) for x in rng.integers(0, (1 << n) - (1 << 20), size=4)] + [(1 << n) - (1 << 20)]
    ranges_d = [dense._copy_range(s0, 1 << 20) for s0 in starts]
    shots_d = L.sample(dense, 2000, rng_seed=5).indices
    dense.release()
    _native.drain_pool()
    sv, rec = L.run_circuit_sharded(circ, L.plan_for_shard_count(n, G), "fp64", memory_budget=budget)
    try:
        kinds = [g.kind for g in rec.gates]
        assert "W" in kinds and "Y" not in kinds, kinds
        red = sv._reductions(None)
        assert red.sum_p == pytest.approx(red_d.sum_p, rel=1e-12)
        assert red.sum_p_cut == pytest.approx(red_d.sum_p_cut, rel=1e-11)
        assert int(red.argmax_cut) == int(red_d.argmax_cut)
        for s0, want in zip(starts, ranges_d):
            assert normwise(sv._copy_range(s0, 1 << 20), want) < 1e-12
        shots = L.sample(sv, 2000, rng_seed=5).indices
        assert int(np.sum(shots != shots_d)) <= 4
    finally:
        sv.release()


def test_distributed_api_with_one_rank_runs_the_single_gpu_engine():
    """run_circuit_distributed under a one-rank process group (torchrun
    --nproc-per-node 1) is the single-GPU engine: results equal run_circuit's."""
    import socket

    import torch.distributed as dist

    from paper_2604_26423_b200.distributed import drain_dist_pool, run_circuit_distributed

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        inst = L.solve_instance(L.generate_instance(16, 5))
        circ = L.build_circuit(inst, L.LrQaoaParams(p=3))
        sv = run_circuit_distributed(circ, "fp64")
        r = sv.exact_expected_r(inst)
        shots = sv.sample(500, 4)
        amps = sv.gather_amps()
        sv.release()
        dense = L.run_circuit(circ, "fp64")
        assert r == L.exact_expected_r(dense, inst)
        np.testing.assert_array_equal(shots.indices, L.sample(dense, 500, rng_seed=4).indices)
        np.testing.assert_array_equal(amps, dense.amps)
        dense.release()
        drain_dist_pool()
    finally:
        dist.destroy_process_group()


def test_streamed_dump_per_shard_round_trips_byte_identically(tmp_path):
    """LQSV dumps written by every shard's thread into its own byte range,
    loaded back into a different shard count and into one device: the same
    bytes every way (reference format engine.py:279-312)."""
    from paper_2604_26423_b200.engine import lqsv_header
    from paper_2604_26423_b200.sharded import load_statevector_sharded

    n = 20
    circ = L.build_circuit(L.generate_instance(n, 5), L.LrQaoaParams(p=2))
    sv, _ = L.run_circuit_sharded(circ, L.plan_for_shard_count(n, 4), "fp64")
    a = tmp_path / "a.lqsv"
    L.save_statevector(sv, a)  # per-shard writers
    want = sv.amps.astype("<c16").tobytes()
    raw = a.read_bytes()
    assert lqsv_header(a)[0] == n and raw[8:] == want
    back = load_statevector_sharded(a, L.plan_for_shard_count(n, 8))
    b = tmp_path / "b.lqsv"
    L.save_statevector(back, b)
    assert b.read_bytes() == raw
    assert back.norm_squared() == pytest.approx(sv.norm_squared(), rel=1e-14)
    dense = L.load_statevector(a, memory_budget=1 << 30)
    c = tmp_path / "c.lqsv"
    L.save_statevector(dense, c)
    assert c.read_bytes() == raw
    np.testing.assert_array_equal(L.sample(back, 500, rng_seed=3).indices, L.sample(dense, 500, rng_seed=3).indices)
    for s in (sv, back, dense):
        s.release()


@pytest.mark.parametrize("n,G,p,prec,dbeta", [(18, 4, 3, "fp64", 0.2), (17, 8, 1, "fp64", 0.9), (26, 2, 3, "fp32", 0.2),
                                              (16, 2, 5, "fp64", 1.2)])
def test_odd_p_final_pass_runs_in_the_swapped_layout(n, G, p, prec, dbeta):
    """An odd p leaves the global and top local qubits swapped; the engine
    makes no restoring remap: the fused final pass (sum p, sum pC, min/max E,
    the histogram) and the sampler work in that layout - the sampler walks
    the (block, rank) segments of the global CDF - and an amplitude read
    makes the remaining remap.  Against the dense engine."""
    inst = L.solve_instance(L.generate_instance(n, 8), limit=n)
    circ = L.build_circuit(L.generate_instance(n, 8), L.LrQaoaParams(p=p, delta_beta=dbeta))
    sv, rec = L.run_circuit_sharded(circ, L.plan_for_shard_count(n, G), prec)
    dense = L.run_circuit(circ, prec)
    try:
        assert all(d.layout() == 1 for d in sv._shards)
        assert sum(g.kind in "YWT" for g in rec.gates) == p
        red, red_d = sv._reductions(None), dense.device_state.reduce()
        tol = 1e-12 if prec == "fp64" else 1e-6
        assert red.sum_p == pytest.approx(red_d.sum_p, rel=tol)
        assert red.sum_p_cut == pytest.approx(red_d.sum_p_cut, rel=tol)
        assert int(red.argmax_cut) == int(red_d.argmax_cut)
        assert red.min_energy == pytest.approx(red_d.min_energy, rel=1e-12)
        assert red.max_energy == pytest.approx(red_d.max_energy, rel=1e-12)
        s_sh = L.sample(sv, 3000, rng_seed=4).indices
        s_de = L.sample(dense, 3000, rng_seed=4).indices
        if prec == "fp64":
            assert int(np.sum(s_sh != s_de)) <= 2
        else:  # 2^26 outcomes of ~1e-8 mass: fp32 rounding moves some CDF boundaries
            assert np.mean(s_sh == s_de) > 0.9
            assert L.approximation_ratio(inst, L.ShotSet(n, s_sh, 4, "noiseless")) == pytest.approx(
                L.approximation_ratio(inst, L.ShotSet(n, s_de, 4, "noiseless")), rel=2e-3)
        d_sh = L.exact_cut_distribution(sv, inst, bins=256)
        d_de = L.exact_cut_distribution(dense, inst, bins=256)
        assert np.max(np.abs(d_sh.probs - d_de.probs)) < (1e-12 if prec == "fp64" else 1e-6)
        # still swapped unless the shards' blocks are smaller than a tile (the
        # sampler then made the remaining remap itself)
        tiny = (n - (G.bit_length() - 1)) - (G.bit_length() - 1) < (12 if prec == "fp64" else 13)
        assert all(d.layout() == (0 if tiny else 1) for d in sv._shards)
        got = sv.amps  # the remaining remap
        assert all(d.layout() == 0 for d in sv._shards)
        assert normwise(got, dense.amps.astype(np.complex128)) < (1e-12 if prec == "fp64" else 3e-6)
        # reductions and samples after the restore are the same
        assert L.exact_expected_r(sv, inst) == pytest.approx(L.exact_expected_r(dense, inst), rel=tol)
        if prec == "fp64":
            np.testing.assert_array_equal(L.sample(sv, 3000, rng_seed=4).indices, s_sh)
    finally:
        sv.release()
        dense.release()
