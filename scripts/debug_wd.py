"""complex64 vs complex128 engine runs (normwise) for plan debugging."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2604_26423_b200 as L  # noqa: E402

for spec in sys.argv[1:]:
    n, p, db = spec.split(",")
    n, p, db = int(n), int(p), float(db)
    circ = L.build_circuit(L.generate_instance(n, 5), L.LrQaoaParams(p=p, delta_beta=db))
    lo = L.run_circuit(circ, "fp32").amps.astype(np.complex128)
    hi = L.run_circuit(circ, "fp64").amps
    d = lo - hi
    print(spec, "normwise", np.linalg.norm(d) / np.linalg.norm(hi))
    bad = np.abs(d) > 1e-3 * np.abs(hi).max()
    print("  bad fraction", bad.mean())
