"""Where the persistent PPE loop (ppe_loop=3) differs from the host-polled one (1): one step of a
small case, differing pressure entries listed (index, fluid / wall, values)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from parity_util import small_cases, gpu_sim  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "db3d_f32"
case = small_cases()[name]
a, b = gpu_sim(case, ppe_loop=1), gpu_sim(case, ppe_loop=3)
for s in range(3):
    ra, rb = a.step(case.dt), b.step(case.dt)
    pa, pb = a.get("PRESSURE"), b.get("PRESSURE")
    d = np.flatnonzero(pa != pb)
    print(f"step {s}: iters {ra.iters} {rb.iters}; n_fluid {case.n_fluid} of {pa.size}; differing {d.size}", flush=True)
    if d.size:
        print("  first:", [(int(i), float(pa[i]), float(pb[i])) for i in d[:8]])
        print("  fluid rows differing:", int((d < case.n_fluid).sum()), " max |diff|", float(np.abs(pa - pb).max()))
        break
