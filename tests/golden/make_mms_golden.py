"""Generate tests/golden/mms_errors.json — BASELINE config 2 (the manufactured
traveling-wave convergence study, validate.hpp:541-597) run by the UNMODIFIED
reference (oracle/_ref) in this container, where the reference exists.

For N = 1..8 on the curved periodic mesh build_wavy_mesh(N, k, k, amp 0.04)
(validate.hpp:99-101) and k = 8, 16, 32, plus crit_convergence's own cartesian
N = 3 set: the L2(h) error at t = 0.2 with cfl 0.4 and the step count.  The GPU
test (tests/test_gpu_configs.py) reruns the same loop through the GPU forcing path
and compares.  Larger k (to 128) cost the single-threaded reference hours per case
at N >= 5, so the committed table stops at 32.

    python tests/golden/make_mms_golden.py
"""
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

CASES = [("wavy", N, k) for N in range(1, 9) for k in (8, 16, 32)] + \
        [("cartesian", 3, k) for k in (8, 16, 32)]


def run(case):
    from oracle import ref
    kind, N, k = case
    m = ref.build_mesh(kind, N, k, k, periodic_x=True, periodic_y=True)
    err, steps = ref.mms_error(m, ref.params(g=9.81), cfl=0.4, t_end=0.2)
    return {"mesh": kind, "degree": N, "k": k, "l2_h": err, "steps": steps}


if __name__ == "__main__":
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        rows = list(ex.map(run, sorted(CASES, key=lambda c: -c[1] * c[2] ** 3)))
    rows.sort(key=lambda r: (r["mesh"], r["degree"], r["k"]))
    out = {"source": "oracle/_ref (unmodified reference, -O3 -DNDEBUG -ffp-contract=off)",
           "wave": {"h0": 2.0, "amp": 0.2, "u0": 0.7, "v0": 0.3, "k": "2 pi", "g": 9.81},
           "cfl": 0.4, "t_end": 0.2, "rows": rows}
    with open(os.path.join(HERE, "mms_errors.json"), "w") as f:
        json.dump(out, f, indent=1)
    for r in rows:
        print(r)
