"""Write tests/golden/oracle_trajectory_cfg{1,2}.npz: the layouts of the
ORACLE's own L-tsNET run (O5 + O6/O7 from the seeded init, oracle C0 P) at
iterations 249, 260 and 499, used by tests/test_gpu_parity.py::
test_grad_parity_oracle_trajectory.  Calls only oracle/ and the seeded input
generators (workloads/); nothing from the CUDA path.  Each file records a
fingerprint of its P and init so the test recomputes when they change.
    python scripts/make_oracle_trajectory.py [cfg ...]"""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from workloads import config_graph, init_layout  # noqa: E402

ITERS = (249, 260, 499)


def fingerprint(P, Y0) -> str:
    h = hashlib.sha256()
    for a in (P["indptr"], P["indices"], P["values"].astype(np.float32), Y0.astype(np.float32)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [1, 2]
    for cfg in cfgs:
        ip, ix = config_graph(cfg)
        P = oracle.build_P(ip, ix, 40.0, seed=0)
        n = P["n"]
        Y0 = init_layout(n, 0)
        out = {}

        def cb(it, Y, vel, gains):
            if it in ITERS:
                out[it] = Y.astype(np.float32)
        oracle.run_layout(Y0, P["indptr"], P["indices"], P["values"].astype(np.float32).astype(np.float64),
                          max(ITERS) + 1, callback=cb)
        path = os.path.join(ROOT, "tests", "golden", f"oracle_trajectory_cfg{cfg}.npz")
        np.savez_compressed(path, fingerprint=np.array(fingerprint(P, Y0)), iters=np.array(ITERS),
                            **{f"Y{it}": out[it] for it in ITERS})
        print(path, os.path.getsize(path), flush=True)


if __name__ == "__main__":
    main()
