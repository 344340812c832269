"""CPU check of the sampled full-size parity method: the oracle run on a window cut from the volume
reproduces the whole-volume oracle exactly inside the region that exact_region() declares safe."""
import numpy as np
import pytest

import oracle as O
import phantoms as P
from helpers import window_oracle


@pytest.mark.parametrize("name,dims", [("C2", (30, 28, 26)), ("C4", (26, 27, 25))])
def test_window_matches_full_volume(name, dims):
    cfg = P.config(name).resized(*dims)
    n = 4
    full = P.generate(cfg)
    uf, qf = O.run_inputs(full, n)
    for point in [(0, 0, 0), (dims[0] - 1, dims[1] - 1, dims[2] - 1), (13, 14, 12), (dims[0] - 1, 3, 12)]:
        reg, ur, qr = window_oracle(cfg, point, n, r=2)
        sl = tuple(slice(a, b) for a, b in reg)
        assert ur.size > 0
        assert np.array_equal(ur, uf[(slice(None),) + sl])
        assert np.array_equal(qr, qf[(slice(None), slice(None)) + sl])
