"""Multi-process NCCL tests of the distributed engine: one process per GPU
(the torchrun layout), torch.distributed (gloo) as the bootstrap only, the
NCCL communicator and the remap transports inside liblrq.so.

They need at least two visible GPUs and skip otherwise (the round's GPU pool
hands out one B200 per call; the same schedule and kernels run on one GPU in
tests/test_gpu_sharded.py through in-process shard groups, and the host
logic of the schedule under gloo in tests/test_dist_cpu.py).  Reference
semantics replaced: run_circuit_sharded / _ShardWorker (sharded.py:202-385),
including the abort of the whole run when one worker fails
(AbortedRunError, sharded.py:328-349; test_sharded.py:148-161).
"""
import multiprocessing as mproc
import os
import socket

import numpy as np
import pytest

import paper_2604_26423_b200 as L
from paper_2604_26423_b200 import _native

pytestmark = pytest.mark.gpu


def _gpus() -> int:
    try:
        from paper_2604_26423_b200.build import build

        build()
        return _native.device_count()
    except Exception:
        return 0


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, p, prec, env, out_path, fail_rank):
    os.environ.update(env)
    os.environ["LOCAL_RANK"] = str(rank)
    os.environ["LOCAL_WORLD_SIZE"] = str(world)
    os.environ["WORLD_SIZE"] = str(world)
    import torch.distributed as dist

    from paper_2604_26423_b200.distributed import drain_dist_pool, run_circuit_distributed

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    result = {}
    try:
        inst = L.solve_instance(L.generate_instance(n, 3), limit=n)
        circ = L.build_circuit(inst, L.LrQaoaParams(p=p, delta_beta=0.9))
        sv = run_circuit_distributed(circ, prec, memory_budget=1 << 40)
        result["mode"] = sv.device_state.remap_mode
        if fail_rank == rank:
            os._exit(3)  # a dead rank: the others must abort, not hang
        other = L.solve_instance(L.generate_instance(n, 9), limit=n)
        try:
            result["r"] = sv.exact_expected_r(inst)
            result["r_other"] = sv.exact_expected_r(other)  # a recompute on every rank
            result["shots"] = sv.sample(3000, rng_seed=1).indices
            amps = sv.gather_amps()
            if rank == 0:
                result["amps"] = amps
            # per-rank streamed LQSV dump and load
            path = out_path + ".lqsv"
            sv.save(path)
            from paper_2604_26423_b200.distributed import load_statevector_distributed
            back = load_statevector_distributed(path)
            result["reload_equal"] = bool(np.array_equal(back.local_amps(), sv.local_amps()))
            back.release()
        except L.AbortedRunError as exc:
            result["aborted"] = str(exc)
        sv.release()
        drain_dist_pool()
    finally:
        if rank == 0 or fail_rank is not None:
            np.save(out_path + f".{rank}.npy", result, allow_pickle=True)
        if fail_rank is None:
            dist.destroy_process_group()


def _run(world, n, p, prec, env, tmp_path, fail_rank=None, timeout=600):
    ctx = mproc.get_context("spawn")
    port = _free_port()
    out = str(tmp_path / "res")
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, p, prec, env, out, fail_rank))
             for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout)
    for pr in procs:
        if pr.is_alive():
            pr.kill()
            pytest.fail("a rank hung")
    return out, [pr.exitcode for pr in procs]


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("transport", ["fused", "peer", "nccl"])
def test_nccl_ranks_match_the_dense_engine(world, transport, tmp_path):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = {"fused": {}, "peer": {"LRQ_FUSED_REMAP": "0"},
           "nccl": {"LRQ_FUSED_REMAP": "0", "LRQ_PEER_REMAP": "0"}}[transport]
    n, p, prec = 18 + (world.bit_length() - 1), 3, "fp64"
    out, codes = _run(world, n, p, prec, env, tmp_path)
    assert codes == [0] * world
    res = np.load(out + ".0.npy", allow_pickle=True).item()
    assert res["mode"] == transport
    inst = L.solve_instance(L.generate_instance(n, 3), limit=n)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=p, delta_beta=0.9))
    dense = L.run_circuit(circ, prec)
    want = dense.amps.astype(np.complex128)
    assert np.linalg.norm(res["amps"] - want) / np.linalg.norm(want) < 1e-12
    assert res["r"] == pytest.approx(L.exact_expected_r(dense, inst), rel=1e-12)
    other = L.solve_instance(L.generate_instance(n, 9), limit=n)
    assert res["r_other"] == pytest.approx(L.exact_expected_r(dense, other), rel=1e-12)
    assert int(np.sum(res["shots"] != L.sample(dense, 3000, rng_seed=1).indices)) <= 2
    assert res["reload_equal"]
    from paper_2604_26423_b200.engine import load_statevector_amps
    n_file, amps = load_statevector_amps(out + ".lqsv")
    assert n_file == n and amps.tobytes() == res["amps"].astype(np.complex128).tobytes()
    dense.release()


def test_dead_rank_aborts_the_run(tmp_path):
    if _gpus() < 2:
        pytest.skip("needs 2 GPUs")
    out, codes = _run(2, 20, 2, "fp64", {"LRQ_DIST_TIMEOUT_S": "30"}, tmp_path, fail_rank=1, timeout=300)
    assert codes[1] == 3
    res = np.load(out + ".0.npy", allow_pickle=True).item()
    assert "aborted" in res and "aborted run" in res["aborted"]
