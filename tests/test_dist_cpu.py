"""CPU tests of the multi-GPU path's host logic with world_size 2 and 4 (gloo).

Each rank runs in its own process and executes the *distributed plan* that
liblrq.so generates (lrq_describe_dist_plan: sweeps, permutation states,
remap points, partial mixer targets) on a numpy shard, with the rank's phase
and cost terms from lrq_dist_terms, remaps as gloo send/recv block
transposes, and the sampler's rank-partitioned inverse CDF.  The gathered
state, <C> and the sampled indices must match the CPU oracle.  This checks
everything of the distributed engine except the kernels themselves (which
the GPU tests check on one device).
"""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lrq_oracle as O
from paper_2604_26423_b200 import _native


def _rx(state, q, h):
    v = state.reshape(-1, 2, 1 << q)
    a0 = v[:, 0, :].copy()
    a1 = v[:, 1, :].copy()
    c, s = np.cos(h), -1j * np.sin(h)
    v[:, 0, :] = c * a0 + s * a1
    v[:, 1, :] = s * a0 + c * a1


def _local_energy(nl, m, f, c):
    z = np.arange(1 << nl, dtype=np.uint64)
    s = 1.0 - 2.0 * ((z[:, None] >> np.arange(nl, dtype=np.uint64)[None, :]) & np.uint64(1)).astype(np.float64)
    return 0.5 * np.einsum("zi,ij,zj->z", s, m, s) + s @ f + c


def _exchange(state, rank, world, g):
    """All-to-all block transpose (local block b <-> rank b's block `rank`),
    executed step by step as liblrq's remap schedule says
    (lrq_describe_remap: XOR-pairwise steps, one partner per step) with gloo
    send/recv in place of the peer-memory swap / NCCL send-recv."""
    nl = int(np.log2(state.size))
    blocks = state.reshape(world, 1 << (nl - g)).copy()
    for partner, mine, theirs, half in _native.describe_remap(world, rank):
        assert theirs == rank and mine == partner and half == (0 if rank < partner else 1)
        send = torch.from_numpy(blocks[mine].view(np.float64).copy())
        recv = torch.empty_like(send)
        ops = [dist.P2POp(dist.isend, send, partner), dist.P2POp(dist.irecv, recv, partner)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        blocks[mine] = recv.numpy().view(np.complex128)
    return blocks.reshape(-1)


def _worker(rank, world, port, n, p, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = world.bit_length() - 1
        nl = n - g
        plan = json.loads(_native.describe_dist_plan(n, g, 16, p))
        K = plan["K"]
        w = O.instance_weights(n, seed)
        betas, gammas = O.ramp(p)
        state = np.full(1 << nl, O.uniform_amplitude(n, "fp64"), dtype=np.complex128)
        remaps = 0
        for sw, (perm, remap_after, target1) in zip(plan["sweeps"], plan["dist"]):
            gr = plan["groups"][sw["group"]]
            phys = lambda i: i if i < gr["m"] else gr["q0"] + i - gr["m"]  # noqa: E731
            all_t = [phys(i) for i in range(K) if (gr["tmask"] >> i) & 1]
            t1 = [phys(i) for i in range(K) if (target1 >> i) & 1] if target1 else all_t
            if sw["beta1"] >= 0:
                for qb in t1:
                    _rx(state, qb, -betas[sw["beta1"]])
            if sw["phase"] >= 0:
                m, f, c = _native.dist_terms(n, g, rank, perm, gammas[sw["phase"]] * w)
                state *= np.exp(-1j * _local_energy(nl, m, f, c))
            if sw["beta2"] >= 0:
                for qb in all_t:
                    _rx(state, qb, -betas[sw["beta2"]])
            if remap_after:
                state = _exchange(state, rank, world, g)
                remaps += 1
        # final pass in the permutation the layers left (an odd p leaves the
        # global and top local qubits swapped; no restoring remap)
        perm = plan["dist"][-1][0]
        m, f, c = _native.dist_terms(n, g, rank, perm, w)
        cut = 0.5 * (float(w.sum()) - _local_energy(nl, m, f, c))
        probs = (state.real ** 2 + state.imag ** 2)
        sums = torch.tensor([probs.sum(), probs @ cut], dtype=torch.float64)
        parts = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, sums)
        # sampler (lrq_sample): the global CDF in index order is a list of
        # contiguous local segments - the whole shard per rank in the
        # identity layout; block b of every rank, b major, in the swapped one
        L = 1 << (nl - g)
        if perm == 0:
            segs = [(r, 0, 1 << nl, r << nl) for r in range(world)]
        else:
            segs = [(r, b * L, L, (b << nl) | (r << (nl - g))) for b in range(world) for r in range(world)]
        mine = [probs[lo:lo + cnt].sum() for (r, lo, cnt, _) in segs if r == rank]
        allm = [torch.zeros(len(mine), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allm, torch.tensor(mine, dtype=torch.float64))
        mass_of, k_of = {}, {}
        for r in range(world):
            k_of[r] = 0
        for (r, lo, cnt, base) in segs:
            mass_of[(r, lo)] = float(allm[r][k_of[r]])
            k_of[r] += 1
        total = sum(mass_of.values())
        u = O.shot_uniforms(1, 2000)
        idx = np.zeros(u.size, dtype=np.int64)
        off = 0.0
        for (r, lo, cnt, base) in segs:
            mass = mass_of[(r, lo)]
            if r == rank:
                cum = off + np.cumsum(probs[lo:lo + cnt])
                for k, x in enumerate(u):
                    if off / total <= x < (off + mass) / total:
                        j = int(np.searchsorted(cum / total, x, side="right"))
                        idx[k] = base + min(j, cnt - 1)
            off += mass
        shots = torch.from_numpy(idx)
        dist.all_reduce(shots)
        if perm == 1:  # lrq_restore_layout: the remaining remap, for the amplitudes
            state = _exchange(state, rank, world, g)
        gathered = [torch.zeros(2 << nl, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(state.view(np.float64).copy()))
        if rank == 0:
            full = np.concatenate([t.numpy().view(np.complex128) for t in gathered])
            q.put((full, float(sum(x[1] for x in parts)), shots.numpy(), remaps))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2604_26423_b200.build import build

    build()


@pytest.mark.parametrize("world,n,p", [(2, 16, 3), (4, 17, 2), (2, 17, 4), (4, 15, 2), (8, 17, 3)])
def test_distributed_plan_emulation_matches_oracle(world, n, p):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = mp.start_processes(_worker, args=(world, _free_port(), n, p, 3, q), nprocs=world, join=False,
                               start_method="spawn")
    full, sum_pc, shots, remaps = q.get()  # before join: the result may exceed the pipe buffer
    procs.join()
    w = O.instance_weights(n, 3)
    want = O.simulate(n, w, p, "fp64")
    assert np.linalg.norm(full - want) / np.linalg.norm(want) < 1e-12
    probs = O.probabilities(want)
    assert sum_pc == pytest.approx(O.expected_cut(n, w, probs), rel=1e-12)
    ref = O.draw(probs, O.shot_uniforms(1, 2000))
    assert int(np.sum(shots.astype(np.uint64) != ref)) <= 1
    assert remaps == p  # one per layer: an odd p's final pass runs in the swapped layout


def test_dist_terms_reproduce_global_energy():
    """The local matrix + field + constant of every rank, in both permutation
    states, reproduce E(z) = sum w s_i s_j of the global index."""
    n, g = 9, 2
    w = O.instance_weights(n, 4)
    z = np.arange(1 << n, dtype=np.uint64)
    s = 1.0 - 2.0 * ((z[:, None] >> np.arange(n, dtype=np.uint64)[None, :]) & np.uint64(1)).astype(np.float64)
    full = O.weight_matrix(n, w)
    e_glob = 0.5 * np.einsum("zi,ij,zj->z", s, full, s)
    nl = n - g
    for perm in (0, 1):
        for rank in range(1 << g):
            m, f, c = _native.dist_terms(n, g, rank, perm, w)
            loc = _local_energy(nl, m, f, c)
            # physical (rank, local) -> logical index under the permutation
            for lz in range(1 << nl):
                bits = [(lz >> k) & 1 for k in range(nl)] + [(rank >> k) & 1 for k in range(g)]
                if perm:
                    bits[nl - g:nl], bits[nl:] = bits[nl:], bits[nl - g:nl]
                zz = sum(b << k for k, b in enumerate(bits))
                assert abs(loc[lz] - e_glob[zz]) < 1e-12


def test_dist_plan_validation():
    with pytest.raises(Exception):
        _native.describe_dist_plan(13, 1, 8, 2)  # n_local must exceed the tile
    plan = json.loads(_native.describe_dist_plan(36, 3, 16, 3))
    kinds = [s["kind"] for s in plan["sweeps"]]
    assert kinds[0] == "P" and kinds[-1] == "Q"
    # 3 layer remaps; the final pass runs in the swapped layout (no 4th remap)
    assert sum(r for _, r, _ in plan["dist"]) == 3 and plan["dist"][-1][0] == 1


@pytest.mark.parametrize("n,g,B,p", [(32, 3, 8, 3), (34, 3, 16, 3), (30, 1, 8, 2), (29, 2, 16, 4), (36, 3, 16, 3)])
def test_dist_plan_remap_follows_group_a_mixer(n, g, B, p):
    """The fused remap redirects the stores of the sweep before a remap; that
    needs a group-A (contiguous-tile) mixer-only sweep there.  Every remap
    has one (an odd p ends in the swapped layout instead of remapping back)."""
    plan = json.loads(_native.describe_dist_plan(n, g, B, p))
    before = [(sw["kind"], plan["groups"][sw["group"]]["kind"])
              for sw, (_, remap_after, _) in zip(plan["sweeps"], plan["dist"]) if remap_after]
    assert len(before) == p  # no restoring remap: the final pass runs in the layout the layers left
    assert all(b == ("M", "A") for b in before)
    assert plan["dist"][-1][0] == p % 2


@pytest.mark.parametrize("B", [8, 16])
@pytest.mark.parametrize("g", [1, 2, 3])
def test_dist_plan_groups_partition_the_local_qubits(g, B):
    """Every n with n_local above the tile is plannable: the groups' mixer
    targets partition the local qubits, and the last group holds the top g
    (the qubits a remap swaps out), taking them from the group below when
    it is short."""
    KA = 13 if B == 8 else 12
    for n in range(KA + g + 1, 40):
        plan = json.loads(_native.describe_dist_plan(n, g, B, 2))
        nl = n - g
        seen = []
        for grp in plan["groups"]:
            for i in range(KA):
                if (grp["tmask"] >> i) & 1:
                    seen.append(i if i < grp["m"] else grp["q0"] + i - grp["m"])
        assert sorted(seen) == list(range(nl)), (n, g, B)
        last = plan["groups"][-1]
        top = {last["q0"] + i - last["m"] for i in range(last["m"], KA) if (last["tmask"] >> i) & 1}
        assert set(range(nl - g, nl)) <= top


@pytest.mark.parametrize("world", [2, 4, 8, 16])
def test_remap_schedule_is_a_symmetric_xor_pairing(world):
    """Every off-diagonal block pair (r, b) is swapped exactly once, in the
    same step on both ranks, and each rank has one partner per step."""
    seen = {}
    for r in range(world):
        steps = _native.describe_remap(world, r)
        assert len(steps) == world - 1
        for k, (partner, mine, theirs, half) in enumerate(steps):
            assert partner == r ^ (k + 1) and mine == partner and theirs == r
            seen[(r, partner)] = (k, half)
    for (r, b), (k, half) in seen.items():
        assert seen[(b, r)][0] == k and seen[(b, r)][1] == 1 - half
    mirror = _native.describe_remap(world, 1, world - 2)
    assert mirror == [[world - 2, -1, -1, 0 if 1 < world - 2 else 1]]


def test_memory_plan_of_the_headline_configs():
    """north_star configs 4 and 5 fit one B200 per rank without a spare
    buffer: n=36 complex128 on 8 GPUs and n=34 complex128 on 2 GPUs hold
    2^33 amplitudes (128 GiB) per GPU plus < 1 GiB of reductions, cost
    matrices and staging, inside 170 GB."""
    for n, world in ((36, 8), (34, 2), (34, 4), (34, 8), (33, 1)):
        m = _native.describe_memory(n, 16, world, 3)
        g = world.bit_length() - 1
        assert m["state"] == 16 << (n - g)
        assert m["other"] < (1 << 30)
        assert m["state"] + m["other"] <= 170e9, (n, world, m)
    # the fused remap's spare buffer only fits at half the state
    m = _native.describe_memory(34, 16, 8, 3)
    assert m["state"] + m["spare"] + m["other"] < 170e9
    m = _native.describe_memory(36, 16, 8, 3)
    assert m["state"] + m["spare"] > 183e9
