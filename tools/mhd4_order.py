"""Convergence of ideal MHD at orders 3 and 4 on the smooth MHD vortex (2D, z-invariant):
32^2 -> 64^2 -> 128^2 to t = 1, mean L1 of rho and of the face Bx vs the exact solution, and
max |div B| h. One JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from tests.test_mhd4_gpu import _vortex  # noqa: E402

res = {}
for order in (3, 4):
    r = [_vortex(n, order) for n in (32, 64, 128)]
    rho, bx = [x[0] for x in r], [x[1] for x in r]
    res[f"o{order}"] = {"l1_rho": rho, "l1_bx": bx, "divb": [x[3] for x in r],
                        "order_rho": [float(np.log2(rho[i] / rho[i + 1])) for i in range(2)],
                        "order_bx": [float(np.log2(bx[i] / bx[i + 1])) for i in range(2)]}
print(json.dumps(res))
