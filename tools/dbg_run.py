import os, sys, subprocess
code = r'''
import sys, numpy as np
sys.path.insert(0, "tests")
import phantoms as P
from helpers import solver_from_inputs
name = sys.argv[1]
cfg = P.config(name) if name == "C1" else P.config(name).resized(64, 48, 40)
inp = P.generate(cfg)
s = solver_from_inputs(inp)
print("kinfo", s.kernel_info())
s.iterate(3)
u, am = s.labeling()
print("ok", name, float(u.sum()))
'''
for lib in sys.argv[1:]:
    for name in ["C1", "C2", "C4", "C5"]:
        env = dict(os.environ, PF_LIB=lib, CUDA_LAUNCH_BLOCKING="1")
        pr = subprocess.run([sys.executable, "-c", code, name], env=env, capture_output=True, text=True, timeout=300)
        print(lib, name, pr.returncode, pr.stdout.strip()[-300:], pr.stderr.strip()[-300:], flush=True)
