"""GPU gate-by-gate execution (circuits that are not LR-QAOA shaped) against
the reference engine's own amplitudes (tests/golden/gates.npz) and its
known answers (test_engine.py:87-90)."""
import numpy as np
import pytest

import paper_2604_26423_b200 as L
from paper_2604_26423_b200 import _native

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _engine():
    from paper_2604_26423_b200.build import build
    build()
    assert _native.device_count() >= 1


@pytest.mark.parametrize("case", range(6))
def test_random_gate_lists_match_reference(golden, case):
    g = golden("gates.npz")
    n, prec = int(g[f"n_{case}"]), str(g[f"prec_{case}"])
    kinds, qa, qb = g[f"gates_{case}"]
    names = ("H", "RX", "RZZ")
    gates = []
    for k, a, b, t in zip(kinds, qa, qb, g[f"theta_{case}"]):
        k = int(k)
        gates.append(L.GateOp(names[k], (int(a),) if k < 2 else (int(a), int(b)), None if k == 0 else float(t)))
    sv = L.run_circuit(L.CircuitIR(num_qubits=n, gates=gates), prec)
    want = g[f"amps_{case}"]
    got = sv.amps
    assert got.dtype == want.dtype
    err = np.abs(got.astype(np.complex128) - want).max()
    assert err <= (1e-13 if prec == "fp64" else 1e-6), err


def test_rzz_pi_on_plus_state_known_answer():
    sv = L.init_plus_state(2, "fp64")
    L.apply_rzz(sv, np.pi, 0, 1)
    np.testing.assert_allclose(sv.amps, [-0.5j, 0.5j, 0.5j, -0.5j], atol=1e-15)


def test_gate_validation_and_reductions():
    sv = L.zero_state(3, "fp64")
    with pytest.raises(L.ValidationError):
        L.apply_h(sv, 3)
    with pytest.raises(L.ValidationError):
        L.apply_rzz(sv, 0.1, 1, 1)
    for q in range(3):
        L.apply_h(sv, q)
    inst = L.solve_instance(L.WmcInstance(3, ((0, 1, 0.5), (0, 2, 1.0), (1, 2, 0.25))))
    # uniform distribution: exact r = (W/2) / C* (the random baseline)
    assert L.exact_expected_r(sv, inst) == pytest.approx(L.random_baseline_expectation(inst), rel=1e-12)
    assert sv.norm_squared() == pytest.approx(1.0, rel=1e-14)


def test_large_state_gate_path_matches_fused_path():
    # an LR-QAOA circuit with one extra gate takes the gate-by-gate path; without
    # it the fused sweeps: the shared prefix agrees to rounding
    inst = L.generate_instance(16, 3)
    circ = L.build_circuit(inst, L.LrQaoaParams(p=2))
    fused = L.run_circuit(circ, "fp64").amps
    extra = L.CircuitIR(num_qubits=16, gates=list(circ.gates) + [L.GateOp("RX", (0,), 0.0)])
    gated = L.run_circuit(extra, "fp64").amps
    assert np.linalg.norm(gated - fused) / np.linalg.norm(fused) < 1e-12


@pytest.mark.parametrize("name,n,seed,p,prec", [("lqsv_n8_fp64.bin", 8, 2, 3, "fp64"), ("lqsv_n9_fp32.bin", 9, 3, 2, "fp32")])
def test_lqsv_load_of_reference_dump_and_round_trip(tmp_path, name, n, seed, p, prec):
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name)
    ref = L.load_statevector(path)
    assert ref.num_qubits == n and ref.precision is L.Precision.coerce(prec)
    mine = L.run_circuit(L.build_circuit(L.generate_instance(n, seed), L.LrQaoaParams(p=p)), prec)
    tol = 1e-12 if prec == "fp64" else 1e-6
    assert np.abs(ref.amps.astype(np.complex128) - mine.amps).max() < tol
    out = tmp_path / "s.bin"
    L.save_statevector(ref, out)
    assert out.read_bytes() == open(path, "rb").read()  # byte-identical dump of the loaded state
    # the loaded state is a live device state: reductions and sampling work on it
    inst = L.solve_instance(L.generate_instance(n, seed))
    assert L.exact_expected_r(ref, inst) == pytest.approx(L.exact_expected_r(mine, inst), rel=1e-5)


@pytest.mark.parametrize("n", [3, 14])
@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_pauli_seams_are_exact(n, dtype):
    """noise._x/_y/_z_kernel and _apply_pauli_pair (the reference's private
    Pauli seams, noise.py:70-98) on the GPU: exact, in place on the host array."""
    from paper_2604_26423_b200 import noise

    rng = np.random.default_rng(n)
    start = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)).astype(dtype)
    z = np.arange(1 << n)

    def pauli(a, k, q):  # numpy restatement by index: X swaps, Y = i X Z, Z flips the sign of bit 1
        bit = (z >> q) & 1
        if k == 1:
            return a[z ^ (1 << q)]
        if k == 2:
            return np.where(bit == 1, 1j, -1j).astype(a.dtype) * a[z ^ (1 << q)]
        return np.where(bit == 1, -1, 1).astype(a.dtype) * a

    for k, fn in ((1, noise._x_kernel), (2, noise._y_kernel), (3, noise._z_kernel)):
        for q in (0, n - 1):
            amps = start.copy()
            fn(amps, q)
            np.testing.assert_array_equal(amps, pauli(start, k, q))
    for code in range(1, 16):
        amps = start.copy()
        noise._apply_pauli_pair(amps, code, 0, n - 1)
        pa, pb = divmod(code, 4)
        want = start
        if pb:
            want = pauli(want, pb, n - 1)
        if pa:
            want = pauli(want, pa, 0)
        np.testing.assert_array_equal(amps, want)
