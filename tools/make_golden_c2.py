"""Writes tests/golden/c2_oracle.npz: O-EXACT fingerprints of BASELINE configs[1] (C2 and C2-cl,
n = 1000, every 10th step of the 200-step drift sequence), computed ONLY by oracle/ (cyclic Jacobi,
oracle/exact.py) on the seeded inputs of workloads/generators.py. The oracle needs ~1 min per matrix
at n = 1000, too slow for the GPU suite, so the suite compares against these stored values:

  w_{cfg}_{t}    all eigenvalues of A_t, descending (Ritz-value parity, R34; sign counts)
  piz_{cfg}_{t}  Pi(A_t) Z for the fixed probe Z = default_rng(20191206).standard_normal((1000, 4)):
                 E ||(Pi_gpu - Pi) Z||_F^2 = 4 ||Pi_gpu - Pi||_F^2 (Gaussian probe), so the stored
                 product estimates the Frobenius error without storing Pi (8 MB per matrix)
  pif_{cfg}_{t}  ||Pi(A_t)||_F,  af_{cfg}_{t} ||A_t||_F

  python tools/make_golden_c2.py [--jobs 8]
"""
import argparse
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

OUT = os.path.join(ROOT, "tests", "golden", "c2_oracle.npz")
PROBE_SEED = 20191206
STEPS = list(range(0, 200, 10))


def probe(n):
    return np.random.default_rng(PROBE_SEED).standard_normal((n, 4))


def one(args):
    name, t, A = args
    from oracle.exact import project_exact
    P, parts = project_exact(A, return_parts=True)
    w = np.sort(parts["w"])[::-1]
    return name, t, w, P @ probe(A.shape[0]), float(np.linalg.norm(P)), float(np.linalg.norm(A))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=os.cpu_count())
    args = ap.parse_args()
    from workloads.generators import C2, C2CL, drift_sequence
    jobs = []
    for cfg in (C2(), C2CL()):
        for t, A, _ in drift_sequence(cfg, steps=cfg.steps):
            if t in STEPS:
                jobs.append((cfg.name, t, A.copy()))
    out = {}
    with ProcessPoolExecutor(max_workers=args.jobs) as ex:
        for name, t, w, pz, pf, af in ex.map(one, jobs):
            key = f"{name.replace('-', '')}_{t}"
            out[f"w_{key}"] = w
            out[f"piz_{key}"] = pz
            out[f"pif_{key}"] = np.array(pf)
            out[f"af_{key}"] = np.array(af)
            print(key, flush=True)
    np.savez_compressed(OUT, **out)
    print(OUT, os.path.getsize(OUT))


if __name__ == "__main__":
    main()
