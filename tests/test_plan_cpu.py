"""CPU tests of the C ABI library surface and of the sweep planner.

* liblrq.so loads and exports every symbol include/lrq.h declares (no GPU
  call is made);
* lrq_describe_plan (host-only) produces plans whose sweeps, executed by a
  numpy emulator of the *plan* (not of the kernels), reproduce the oracle's
  final state — this checks the ping-pong ordering, the fused
  mix->phase->mix sweeps, group coverage and round masks without a GPU.
"""
import json
import os
import re

import numpy as np
import pytest

from oracle import lrq_oracle as O
from paper_2604_26423_b200 import _native
from paper_2604_26423_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build()
    return _native.lib()


def test_library_exports_every_header_symbol(lib):
    header = open(os.path.join(ROOT, "include", "lrq.h")).read()
    declared = set(re.findall(r"\b(lrq_[a-z_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    missing = [name for name in sorted(declared) if not hasattr(lib, name)]
    assert not missing, missing
    assert declared == set(_native.EXPORTED)
    assert lib.lrq_abi_version() == _native.ABI_VERSION


def test_describe_plan_validation(lib):
    with pytest.raises(Exception):
        _native.describe_plan(10, 12, 3)
    with pytest.raises(Exception):
        _native.describe_plan(10, 8, 0)


def _rx(state, q, h):
    v = state.reshape(-1, 2, 1 << q)
    a0 = v[:, 0, :].copy()
    a1 = v[:, 1, :].copy()
    c, s = np.cos(h), -1j * np.sin(h)
    v[:, 0, :] = c * a0 + s * a1
    v[:, 1, :] = s * a0 + c * a1


def _energy(n, coeffs):
    z = np.arange(1 << n, dtype=np.uint64)
    e = np.zeros(1 << n)
    k = 0
    for i in range(n):
        si = 1.0 - 2.0 * ((z >> np.uint64(i)) & np.uint64(1)).astype(np.float64)
        for j in range(i + 1, n):
            sj = 1.0 - 2.0 * ((z >> np.uint64(j)) & np.uint64(1)).astype(np.float64)
            e += coeffs[k] * si * sj
            k += 1
    return e


def emulate(plan, n, phase, mixer):
    """Execute a plan's sweep semantics on a dense numpy state."""
    state = np.full(1 << n, O.uniform_amplitude(n, "fp64"), dtype=np.complex128)
    K = plan["K"]
    groups = plan["groups"]
    applied = np.zeros((len(mixer), n), dtype=int)
    for sw in plan["sweeps"]:
        g = groups[sw["group"]]
        m, q0, tmask = g["m"], g["q0"], g["tmask"]
        targets = [i if i < m else q0 + i - m for i in range(K) if (tmask >> i) & 1]
        if g.get("cross", -1) >= 0:  # cluster group: the qubit between the two CTAs' half tiles
            targets.append(g["cross"])
        assert all(0 <= q < n for q in targets)
        if sw["beta1"] >= 0:
            for q in targets:
                _rx(state, q, mixer[sw["beta1"]])
                applied[sw["beta1"], q] += 1
        if sw["phase"] >= 0:
            assert applied[sw["phase"] - 1].min() == 1 if sw["phase"] > 0 else True
            assert applied[sw["phase"]].max() == 0
            state *= np.exp(-1j * _energy(n, phase[sw["phase"]]))
        if sw["beta2"] >= 0:
            for q in targets:
                _rx(state, q, mixer[sw["beta2"]])
                applied[sw["beta2"], q] += 1
    assert np.all(applied == 1), "every layer must mix every qubit exactly once"
    return state


@pytest.mark.parametrize("n,p,pb", [(13, 1, 8), (14, 3, 8), (16, 2, 16), (17, 3, 8), (18, 4, 16),
                                    (20, 3, 8), (23, 2, 8), (24, 3, 16), (21, 5, 16)])
def test_plan_emulation_matches_oracle(lib, n, p, pb):
    plan = json.loads(_native.describe_plan(n, pb, p))
    assert not plan["small"]
    w = O.instance_weights(n, 3)
    betas, gammas = O.ramp(p)
    phase = np.array([[g * x for x in w] for g in gammas])
    mixer = np.array([-b for b in betas])  # RX(theta=-2 beta): half angle -beta
    if n > 20:  # emulation only (oracle too slow): check structure
        S = len(plan["groups"])
        assert len(plan["sweeps"]) == (1 + p * (S - 1) if S > 1 else p + (p == 1))
        return
    got = emulate(plan, n, phase, mixer)
    want = O.simulate(n, w, p, "fp64")
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12


@pytest.mark.parametrize("n", [12, 13, 20, 26, 30, 32, 33, 34, 36])
@pytest.mark.parametrize("pb", [8, 16])
def test_plan_structure(lib, n, pb):
    for p in (1, 2, 3, 10):
        plan = json.loads(_native.describe_plan(n, pb, p))
        K = plan["K"]
        if n < K:
            assert plan["small"]
            continue
        groups = plan["groups"]
        # groups partition the qubits
        cover = []
        for g in groups:
            cover += [i if i < g["m"] else g["q0"] + i - g["m"] for i in range(K) if (g["tmask"] >> i) & 1]
            if g.get("cross", -1) >= 0:
                cover.append(g["cross"])
                assert g["kind"] in ("C10", "C9", "C8") and pb == 8 and g["cross"] == g["q0"] + K - g["m"]
        assert sorted(cover) == list(range(n))
        S = len(groups)
        sweeps = plan["sweeps"]
        assert len(sweeps) == (1 + p * (S - 1) if S > 1 else p + (p == 1))
        assert sweeps[0]["init"] and sweeps[0]["phase"] == 0
        assert sweeps[-1]["reduce"] and sweeps[-1]["group"] == 0
        pair = plan["pair"]
        for sw in sweeps:
            g = groups[sw["group"]]
            m1 = m2 = 0
            for lo, a, b, _, _ in sw["rounds"]:
                assert lo in ((2, 7) if sw.get("prog") in (1, 2) else (0, 2, 3, 4, 8))
                assert not (m1 & a) and not (m2 & b), "a target takes one butterfly per mixer"
                m1 |= a
                m2 |= b
            if sw["beta1"] >= 0:
                assert m1 == g["tmask"]
            if sw["beta2"] >= 0:
                assert m2 == g["tmask"]
            # global I/O layouts: lanes walk contiguous units (never the lo=0
            # layout of group A; H layouts keep register units above the run)
            if sw.get("prog") == 1:
                # warp-decoupled high-group sweep (TMA in / out)
                assert g["kind"] != "A" and sw["kind"] in "PMF" and (pair == 1 or g["kind"] == "H")
                continue
            if sw.get("prog") == 2:
                # cluster-pair sweep (every sweep of a cluster group)
                assert g["kind"] in ("C10", "C9", "C8") and sw["kind"] in "PMF"
                continue
            assert g.get("cross", -1) < 0
            for lo in {sw["rounds"][-1][0], sw["rounds"][0][0]}:
                if g["kind"] == "A":
                    assert lo != 0
                else:
                    assert lo >= g["m"] - pair
        if n in (32,) and pb == 8:
            assert S == 3  # 2 HBM passes per layer for the bench workload


@pytest.mark.parametrize("n", [29, 30, 31, 32, 33])
def test_cluster_plan_structure(lib, n, monkeypatch):
    """The opt-in cluster plan (LRQ_CLUSTER=1): group A plus two C groups of
    8-10 targets (128 KB pair tiles, 128-512 B runs); every sweep of a C
    group runs the cluster-pair kernel (prog 2); the cross qubit is the
    group's top target."""
    monkeypatch.setenv("LRQ_CLUSTER", "1")
    plan = json.loads(_native.describe_plan(n, 8, 3))
    groups = plan["groups"]
    assert [g["kind"][0] for g in groups] == ["A", "C", "C"]
    cover = []
    for g in groups:
        cover += [i if i < g["m"] else g["q0"] + i - g["m"] for i in range(13) if (g["tmask"] >> i) & 1]
        if g["cross"] >= 0:
            cover.append(g["cross"])
            assert g["m"] == 14 - int(g["kind"][1:]) and g["cross"] == g["q0"] + 13 - g["m"]
    assert sorted(cover) == list(range(n))
    assert groups[1]["m"] <= groups[2]["m"]  # the longer runs on the top qubits
    for sw in plan["sweeps"]:
        assert (sw["prog"] == 2) == (sw["group"] != 0)
    if n == 32:
        assert [g["kind"] for g in groups] == ["A", "C10", "C9"]
    monkeypatch.setenv("LRQ_CLUSTER", "0")
    assert all(g["cross"] < 0 for g in json.loads(_native.describe_plan(n, 8, 3))["groups"])
