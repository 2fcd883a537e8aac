import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from parity_util import gpu_sim, oracle_from_gpu  # noqa: E402

case = synth.hydrostatic(nx=40, ny=80, dx=0.025, precision=64)
sim = gpu_sim(case)
o = oracle_from_gpu(case, sim)
w = case.tag == 1
ng, no = sim.get("NORMAL")[w], o.get("normal")[w]
x = case.x[w]
bad = np.abs(ng - no).max(1) > 1e-8
print("bad", bad.sum(), "of", w.sum())
for i in np.flatnonzero(bad)[:30]:
    print(x[i] / case.dx, ng[i], no[i])
