"""Diagnose GPU-vs-oracle drift for SHIFT_NONE on DAG graphs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle as O
import phantoms as P
from helpers import solver_from_inputs
for name, dims in (("C3", (33, 17, 9)), ("C4", (35, 70, 21))):
    inp = P.generate(P.config(name).resized(*dims))
    s = solver_from_inputs(inp, shift=1)
    ur, qr = O.init_state(6, 9, inp.shape, 3)
    t = 0
    for n in (1, 2, 5, 10, 20, 50, 100, 150, 200, 300):
        s.iterate(n - t); O.run_inputs(inp, n - t, shift=1, state=(ur, qr)); t = n
        u, _ = s.labeling(); q = s.flows()
        du = np.abs(u - ur); dq = np.abs(q - qr)
        i = np.unravel_index(np.argmax(du), du.shape)
        print(name, n, "du", du.max(), "at", i, "dq", dq.max(), "umax", ur.max(), flush=True)
