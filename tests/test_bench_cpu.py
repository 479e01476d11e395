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
