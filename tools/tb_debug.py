"""Debug helper: where does a tblock = 2 solver differ from tblock = 0 after n iterations?"""
import sys
import numpy as np
sys.path.insert(0, "tests")
import phantoms as P
from helpers import solver_from_inputs

def cfg(K, dims, sfield=True):
    nx, ny, nz = dims
    return P.Config(f"T{K}", 2 if nz == 1 else 3, nx, ny, nz, "potts", K, 4 * K, 0.15, "sq", "edge" if sfield else "scalar",
                    0.05 if sfield else 0.1, 300, seed=2020)

import os
CK = int(os.environ.get("CK", "0"))
for K, dims, n, sf in [(2, (30, 20, 10), 4, True), (2, (30, 20, 10), 6, False), (3, (30, 20, 1), 4, False),
                       (2, (60, 20, 10), 2, True), (2, (60, 20, 10), 4, True), (2, (60, 20, 10), 20, True)]:
    inp = P.generate(cfg(K, dims, sf))
    a = solver_from_inputs(inp, check_every=CK)
    b = solver_from_inputs(inp, tblock=2, check_every=CK)
    a.iterate(n); b.iterate(n)
    ua, _ = a.labeling(); ub, _ = b.labeling()
    qa = a.flows(); qb = b.flows()
    print(K, dims, n, "sfield", sf, "tb chunk", b.kernel_info())
    du = np.abs(ua - ub).max(0)
    dq = np.abs(qa - qb).max(axis=(0, 1))
    for name, d in (("u", du), ("q", dq)):
        bad = np.argwhere(d > 0)
        print(f"  {name}: max {d.max():.3g}, {len(bad)} voxels differ")
        if len(bad):
            zz, yy, xx = bad[:, 0], bad[:, 1], bad[:, 2]
            print("   z:", np.unique(zz)[:20], " y:", np.unique(yy)[:20], " x:", np.unique(xx)[:40])
    # per component of q
    for k in range(qa.shape[1]):
        d = np.abs(qa[:, k] - qb[:, k]).max()
        print(f"   q comp {k}: {d:.3g}")
