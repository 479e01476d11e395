"""Golden files of the reference CLI (run in the build container, where the
reference package is importable):

    cli_n12_inst.json  lrqbench gen --n 12 --seed 7
    cli_n12_res.json   lrqbench simulate --instance cli_n12_inst.json --p 3
                       --precision fp64 --shots 1000 --seed 1
"""
import os
import shutil
import sys
import tempfile

sys.path.insert(0, "/root/reference/pkg/src")
from lrqbench.cli import main  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

with tempfile.TemporaryDirectory() as d:
    inst, res = os.path.join(d, "i.json"), os.path.join(d, "r.json")
    assert main(["gen", "--n", "12", "--seed", "7", "--out", inst]) == 0
    assert main(["simulate", "--instance", inst, "--out", res, "--p", "3", "--precision", "fp64",
                 "--shots", "1000", "--seed", "1"]) == 0
    shutil.copy(inst, os.path.join(HERE, "cli_n12_inst.json"))
    shutil.copy(res, os.path.join(HERE, "cli_n12_res.json"))
