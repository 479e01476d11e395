"""The bench.py contract pieces that run without a GPU: the reference arm's
JSON line (keys, units, e2e with zero transfer bytes) on a tiny budget, and
the launch accounting behind `gpu_launches`."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--n", "20", "--p", "2", "--cpu-seconds", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["metric"] == "LR-QAOA layer amplitude-updates/s" and line["unit"] == "amp-updates/s"
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["e2e"]["value"] == line["value"] and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] in ("port", "reference") and line["cpu_baseline"]["cores"] >= 1


def test_kernel_launch_accounting():
    import bench
    # P, M, F, M, R sweeps + one-CTA finalize; a fused remap ('Y') and an
    # exchanged one ('T') launch none of our kernels; a flip reversal two
    assert bench.kernel_launches("PMFMRZ", 24) == 6
    assert bench.kernel_launches("PMYFMTQZ", 24) == 6
    assert bench.kernel_launches("PMFMRXZ", 24) == 8
    assert bench.kernel_launches("PMFMRZ", 32) == 5 + 3  # multi-CTA finalize from 8192 tiles


def test_workloads_follow_the_baseline_configs():
    import argparse

    import bench

    def wl(world, **kw):
        a = argparse.Namespace(config=0, n=0, p=0, precision="", shots=0)
        for k, v in kw.items():
            setattr(a, k, v)
        return bench.workload(a, world)

    assert wl(1)[:4] == (32, 10, "fp32", 1000)          # configs[2]: the metric's config
    assert wl(2)[:4] == (34, 3, "fp64", 10000)          # configs[3] over 2 GPUs
    assert wl(8)[:4] == (36, 3, "fp64", 10000)          # configs[4]: the north-star target
    assert wl(1, config=4)[:4] == (33, 3, "fp64", 10000)  # largest one-GPU point of configs[3]
    assert wl(1, config=2)[:4] == (26, 3, "fp64", 1000)
    assert wl(8)[5] == "weak"                            # 2^33 amplitudes per GPU at every N
    assert wl(8, config=4)[5] == "strong" and wl(2, config=4)[5] == "strong"  # n=34 fixed


def test_per_kernel_roofline_accounting():
    import bench

    labels = [("P(H4)", "sweep_wd_kernel"), ("M(A)", "sweep_kernel"), ("F(H)", "sweep_wd_kernel"),
              ("R(A)", "sweep_kernel")]
    # two runs: sweeps plus a finalize record 'Z' each
    ms = [9.0, 11.0, 20.0, 17.0, 0.1, 9.0, 11.0, 20.0, 17.0, 0.1]
    kinds = "PMFRZPMFRZ"
    pk = bench.per_kernel(ms, kinds, labels, 32, 8, 6553.3, 2)
    st = 8 << 32
    assert pk["P(H4)"]["bytes_per_launch"] == st and pk["M(A)"]["bytes_per_launch"] == 2 * st
    assert pk["F(H)"]["launches_per_step"] == 1
    assert abs(pk["M(A)"]["achieved_GBps"] - 2 * st / 11e-3 / 1e9) < 0.1
    assert abs(sum(v["time_share"] for v in pk.values()) - 1.0) < 1e-3
    k, d = bench.dominant(pk, 6553.3)
    assert k == "sweep_wd_kernel" and d["labels"] == ["F(H)", "P(H4)"]
    assert abs(d["achieved"] - 3 * st / 29e-3 / 1e9) < 0.1  # (P bytes + F bytes) / (9 + 20 ms)
