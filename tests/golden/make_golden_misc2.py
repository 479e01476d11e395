"""Reference outputs for host formats (run where the reference is importable):
circuit_n5.txt (circuit_to_text), lqsv_n8_fp64.bin / lqsv_n9_fp32.bin
(save_statevector of a reference run_circuit)."""
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from lrqbench import LrQaoaParams, build_circuit, circuit_to_text, generate_instance, run_circuit, save_statevector  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
circ = build_circuit(generate_instance(5, 1), LrQaoaParams(p=2))
open(os.path.join(HERE, "circuit_n5.txt"), "w").write(circuit_to_text(circ))
save_statevector(run_circuit(build_circuit(generate_instance(8, 2), LrQaoaParams(p=3)), "fp64"),
                 os.path.join(HERE, "lqsv_n8_fp64.bin"))
save_statevector(run_circuit(build_circuit(generate_instance(9, 3), LrQaoaParams(p=2)), "fp32"),
                 os.path.join(HERE, "lqsv_n9_fp32.bin"))
