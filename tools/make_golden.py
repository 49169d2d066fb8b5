"""Write oracle-only reference values for the full-size GPU parity tests.

Calls nothing but ``oracle/`` and ``helm_inputs`` (no CUDA path involved), so
every stored value is an oracle value.  For each config:
  * one double-sweep apply per direction on a seeded random r, sampled at
    seeded node indices;
  * the selective MPGMRES solve (tol 1e-6, x0 = 0): iteration count, residual
    history, true residual, and x at the same sampled nodes.

    python tools/make_golden.py 4 5        # configs to (re)generate
Output: tests/golden/oracle_C<k>.npz
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from helm_inputs import make_config, random_vector
from oracle import krylov, p1, sweep

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
NSAMPLE = 512


def main(nums):
    for num in nums:
        t0 = time.time()
        cfg = make_config(num)
        A = p1.assemble(cfg)
        b = p1.load_vector(cfg)
        rng = np.random.default_rng(5000 + num)
        idx = np.sort(rng.choice(cfg.n, size=min(NSAMPLE, cfg.n), replace=False))
        precs = [sweep.make_preconditioner(cfg, A, nm) for nm in cfg.dirs]
        t1 = time.time()
        r = random_vector(cfg.n, 900 + num)
        z_samples = np.stack([P.apply(r)[idx] for P in precs])
        t2 = time.time()
        x, st = krylov.mpgmres(A, [P.apply for P in precs], b, tol=cfg.tol, maxit=cfg.maxit)
        t3 = time.time()
        np.savez_compressed(os.path.join(OUT, f"oracle_{cfg.name}.npz"), idx=idx, r_seed=900 + num,
                            dirs=np.array(cfg.dirs), z=z_samples, x=x[idx], iterations=st.iterations,
                            history=np.array(st.history), true_rel_res=st.true_rel_res,
                            b_norm=np.linalg.norm(b), x_norm=np.linalg.norm(x))
        print(f"{cfg.name}: setup {t1-t0:.1f}s apply x{len(precs)} {t2-t1:.1f}s solve {t3-t2:.1f}s "
              f"iterations {st.iterations} true_rel_res {st.true_rel_res:.3e}", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5])
