"""Write tests/golden/matvec_<cfg>.npz: oracle direct sums on BJ's matvec parity protocol
(north_star: "above 10^5 points, matvecs are checked against the direct sum on 4096 seeded
random target rows"; SURVEY.md §8(d) parity protocol).

For each config: both directions (K v: targets x, sources y; K^T u: targets y, sources x), both
kernels (0: exp(-lam c), 1: c exp(-lam c)), weights (i) the marginals b / a and (ii) seeded
U(0,1) (synthetic.uniform_test_weights), on the seeded rows synthetic.check_rows(ci, 4096, ...)
(seed 0 for x rows, seed 1 for y rows). Weights (iii), the GPU's own converged iterate, cannot be
precomputed; tests/test_gpu_parity.py evaluates the oracle on them at test time.

Calls only oracle/ (oracle.dense.direct_sum: Eq. (matexp)/(matexpt) P:L462-470, Neumaier sums)
and the synthetic input generators. Long-running (c5: about an hour on 8 cores):

    nice python tools/make_golden_matvec.py c3 c4 c5
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import dense  # noqa: E402
from synthetic import check_rows, get, make_inputs, uniform_test_weights  # noqa: E402
from synthetic.configs import CONFIG_INDEX  # noqa: E402

ROWS = 4096


def path(name):
    return os.path.join(ROOT, "tests", "golden", f"matvec_{name}.npz")


def main(names):
    for name in names:
        cfg = get(name)
        ci = CONFIG_INDEX[name]
        t0 = time.time()
        x, y, a, b = make_inputs(cfg)
        rx = check_rows(ci, ROWS, x.shape[0])
        ry = check_rows(ci, ROWS, y.shape[0], seed=1)
        weights = {"marginal": (b, a),
                   "uniform01": (uniform_test_weights(ci, y.shape[0]), uniform_test_weights(ci, x.shape[0], 1))}
        out = {"rows_x": rx, "rows_y": ry}
        for wname, (wy, wx) in weights.items():
            for kernel in (0, 1):
                out[f"t_{wname}_k{kernel}"] = dense.direct_sum(x, y, wy, cfg.lam, kernel, rows=rx)
                out[f"tt_{wname}_k{kernel}"] = dense.direct_sum(y, x, wx, cfg.lam, kernel, rows=ry)
                print(name, wname, kernel, f"{time.time() - t0:.0f}s", flush=True)
        meta = {"config": name, "n": int(x.shape[0]), "m": int(y.shape[0]), "rows": ROWS,
                "oracle_seconds": time.time() - t0, "oracle_threads": dense.num_threads(),
                "source": "tools/make_golden_matvec.py -> oracle.dense.direct_sum (Eq. (matexp)/(matexpt) "
                          "P:L462-470); t = K w on rows_x (targets x, sources y), tt = K^T w on rows_y"}
        np.savez_compressed(path(name), meta=np.array(json.dumps(meta)), **out)
        print(name, meta, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c3", "c4", "c5"])
