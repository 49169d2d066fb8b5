"""Oracle FD5 (paper-calibration mode) against the paper's Table 1:
h = 2^-9, N = 8, k in {50, 100, 200}; LRL, LRL+BTB, LR+RL, LR+BT+RL+TB with
the "recent" (P:L93 literal) and "core" gathers.  CPU only, oracle only; about
10 minutes per (k, gather) on one core.   python tools/fd5_tables.py [k ...]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from helm_inputs import HelmConfig
from oracle import fd5, krylov, sweep

PAPER = {50.0: [20, 9, 31, 18], 100.0: [18, 8, 29, 18], 200.0: [17, 9, 31, 18]}
COMBOS = (["LRL"], ["LRL", "BTB"], ["LR", "RL"], ["LR", "BT", "RL", "TB"])


def cfg_fd5(e, k, N=8):
    n = 2 ** e
    c = np.ones((n + 1, n + 1))
    return HelmConfig(f"fd5_h{e}_k{k}", n, n, 1.0, 1.0, k, c, np.zeros_like(c, np.complex128), N, 1, ["LRL", "BTB"])


if __name__ == "__main__":
    ks = [float(a) for a in sys.argv[1:]] or [50.0, 100.0, 200.0]
    for k in ks:
        cfg = cfg_fd5(9, k)
        A = fd5.assemble(cfg)
        b = fd5.source(cfg)
        for gather in ("recent", "core"):
            t0 = time.time()
            names = ["LRL", "BTB", "LR", "RL", "BT", "TB"]
            P = dict(zip(names, sweep.make_preconditioners(cfg, A, names, gather=gather, disc="fd5")))
            its = []
            for combo in COMBOS:
                _, st = krylov.mpgmres(A, [P[n].apply for n in combo], b, tol=1e-6, maxit=120)
                its.append(st.iterations)
            print(f"k={k:g} gather={gather}: LRL / LRL+BTB / LR+RL / LR+BT+RL+TB = {its}  "
                  f"(paper {PAPER.get(k)}; {time.time() - t0:.0f} s)", flush=True)
