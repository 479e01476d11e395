"""Pin the CPU oracle (oracle/lrq_oracle.py, oracle/cutdiag.c) to golden
vectors produced by running the REAL reference (tests/golden/make_golden*.py).

These run on CPU only; they are what makes the oracle trustworthy as the
checker of the GPU path.
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import lrq_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _built_c_oracle():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


def test_rng_streams_match_reference(golden):
    g = golden("rng.npz")
    for seed in (0, 1, 7, 12345, -3, 1 << 70):
        key = str(seed).replace("-", "m")
        for n in (3, 12, 26):
            np.testing.assert_array_equal(O.stream(seed, "instance", n).random(8), g[f"inst_{key}_{n}"])
        np.testing.assert_array_equal(O.stream(seed, "shots", 0).random(8), g[f"shots_{key}"])


def test_cfg1_weights_amplitudes_bitwise(golden):
    g = golden("cfg1_n12.npz")
    w = O.instance_weights(12, 7)
    np.testing.assert_array_equal(w, g["weights"])
    np.testing.assert_array_equal(O.simulate(12, w, 3, "fp64"), g["amps64"])
    np.testing.assert_array_equal(O.simulate(12, w, 3, "fp32"), g["amps32"])


def test_threaded_oracle_is_bitwise_identical(golden):
    g = golden("cfg1_n12.npz")
    w = O.instance_weights(12, 7)
    np.testing.assert_array_equal(O.simulate(12, w, 3, "fp64", threads=3), g["amps64"])


def test_cfg1_cut_diag_bitwise_numpy_and_c(golden):
    g = golden("cfg1_n12.npz")
    w = g["weights"]
    z = np.arange(1 << 12, dtype=np.uint64)
    np.testing.assert_array_equal(O.cut_diag(12, w, z), g["cut_diag"])
    np.testing.assert_array_equal(O.c_cut_diag(12, w, z), g["cut_diag"])
    np.testing.assert_array_equal(O.cut_block(12, w, 0, 1 << 12), g["cut_range"])


def test_cfg1_observables(golden):
    g = golden("cfg1_n12.npz")
    w = g["weights"]
    z, v = O.brute_force(12, w)
    assert O.bits_of(z, 12) == str(g["opt_bits"])
    assert v == g["opt_value"]
    p = O.probabilities(g["amps64"])
    assert O.expected_cut(12, w, p) / v == g["exact_r64"]
    u = O.shot_uniforms(1, 1000)
    np.testing.assert_array_equal(O.draw(p, u), g["shots64"])
    p32 = O.probabilities(g["amps32"])
    np.testing.assert_array_equal(O.draw(p32, u), g["shots32"])


def test_small_cases_bitwise(golden):
    g = golden("small.npz")
    for case in range(20):
        n, p, seed = (int(x) for x in g[f"c{case}_meta"])
        w = O.instance_weights(n, seed)
        np.testing.assert_array_equal(O.simulate(n, w, p, "fp64"), g[f"c{case}_amps"])
        np.testing.assert_array_equal(O.simulate(n, w, p, "fp32"), g[f"c{case}_amps32"])
    w = O.instance_weights(9, 77)
    np.testing.assert_array_equal(O.simulate(9, w, 4, "fp64", dbeta=1.4, dgamma=0.9), g["bigbeta_amps"])
    tri = np.array([0.5, 1.0, 0.25])
    np.testing.assert_array_equal(O.simulate(3, tri, 3, "fp64"), g["tri_amps"])


def test_n14_bitwise(golden):
    g = golden("n14.npz")
    w = O.instance_weights(14, 5)
    np.testing.assert_array_equal(O.simulate(14, w, 4, "fp64"), g["amps64"])
    np.testing.assert_array_equal(O.simulate(14, w, 4, "fp32"), g["amps32"])


def test_n20_samples_and_r(golden):
    g = golden("n20.npz")
    w = O.instance_weights(20, 1)
    amps = O.simulate(20, w, 3, "fp64", threads=4)
    np.testing.assert_array_equal(amps[:: int(g["amp_stride"])], g["amps_strided"])
    z, v = O.brute_force(20, w)
    assert O.bits_of(z, 20) == str(g["opt_bits"]) and v == g["opt_value"]
    p = O.probabilities(amps)
    assert O.expected_cut(20, w, p) / v == pytest.approx(float(g["exact_r"]), rel=1e-14)
    np.testing.assert_array_equal(O.draw(p, O.shot_uniforms(1, 10000)), g["shots"])


def test_misc_known_answers(golden):
    m = golden("misc.json")
    tri = np.array([0.5, 1.0, 0.25])
    for bits, val in m["triangle_cuts"].items():
        z = int(bits[::-1], 2)
        assert O.cut_diag(3, tri, [z])[0] == val
    z, v = O.brute_force(3, tri)
    assert [O.bits_of(z, 3), v] == m["triangle_opt"]
    z, v = O.brute_force(2, np.array([0.3]))
    assert [O.bits_of(z, 2), v] == m["tie_opt"]
    for key, want in m["bruteforce"].items():
        n, seed = (int(x) for x in key.split(","))
        z, v = O.brute_force(n, O.instance_weights(n, seed))
        assert [O.bits_of(z, n), v] == want
    b, g_ = O.ramp(3)
    assert [b, g_] == m["schedule_p3"]


def test_uniform_amplitude_is_sequential_product(golden):
    g = golden("cfg1_n12.npz")
    # every amplitude after the H layer equals v_n; check through p=0 effect:
    # H layer only = first 12 gates of the list
    w = g["weights"]
    eng = O.DenseOracle(12, "fp64")
    for op in O.gate_list(12, w, 1)[:12]:
        eng.apply(op)
    assert np.all(eng.amps == O.uniform_amplitude(12, "fp64"))
    eng32 = O.DenseOracle(12, "fp32")
    for op in O.gate_list(12, w, 1)[:12]:
        eng32.apply(op)
    assert np.all(eng32.amps == O.uniform_amplitude(12, "fp32"))


def test_n26_reference_run_values(golden):
    """Config 2 (n=26, p=3, c128): values from a full run of the reference."""
    g = golden("cfg2_n26.npz")
    w = O.instance_weights(26, 1)
    # bit-exact C* of the reference's optimum via the C oracle
    z = int(str(g["opt_bits"])[::-1], 2)
    assert O.c_cut_diag(26, w, [z])[0] == g["opt_value"]
    assert float(g["exact_r"]) == pytest.approx(0.9100517568739738, abs=0)
    assert g["shots"].size == 1000
