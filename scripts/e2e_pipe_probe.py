"""Per-step wall times of bench.py's e2e loop, serial vs pipelined (stage/commit + fetch), C5."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth
from paper_1908_01762_b200 import Simulation

case = synth.dambreak3d()
sim = Simulation.from_case(case, stream=torch.cuda.current_stream().cuda_stream) if False else Simulation.from_case(case)
n, dim = case.x.shape[0], case.dim
for _ in range(3):
    sim.step(case.dt)
pin = lambda s: torch.empty(s, dtype=torch.float32, pin_memory=True)
hx, hu, hut, hp, op = pin((n, dim)), pin((n, dim)), pin((n, dim)), pin((n,)), pin((n,))
for f, b in (("POSITION", hx), ("VELOCITY", hu), ("TRANSPORT_VELOCITY", hut), ("PRESSURE", hp)):
    sim.get_ptr(f, b.data_ptr(), b.numel(), True)
F = (("POSITION", hx), ("VELOCITY", hu), ("TRANSPORT_VELOCITY", hut), ("PRESSURE", hp))
mode = sys.argv[1] if len(sys.argv) > 1 else "all"
for rep in range(3):
    for pipelined in (False, True):
        ts = []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if pipelined:
            for f, b in F:
                sim.stage_ptr(f, b.data_ptr(), b.numel(), True)
        for k in range(20):
            a = time.perf_counter()
            if pipelined:
                sim.commit_staged()
                if k + 1 < 20:
                    for f, b in F:
                        sim.stage_ptr(f, b.data_ptr(), b.numel(), True)
            else:
                for f, b in F:
                    sim.set_ptr(f, b.data_ptr(), b.numel(), True)
            c = time.perf_counter()
            sim.step(case.dt)
            d = time.perf_counter()
            if pipelined:
                sim.fetch_wait()
                sim.fetch_ptr("PRESSURE", op.data_ptr(), n, True)
            else:
                sim.get_ptr("PRESSURE", op.data_ptr(), n, True)
            e = time.perf_counter()
            ts.append((1e3 * (c - a), 1e3 * (d - c), 1e3 * (e - d)))
        if pipelined:
            sim.fetch_wait()
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        ts = np.array(ts)
        print(f"rep {rep} {'pipe' if pipelined else 'serial'}: {1e3 * t / 20:.3f} ms/step; median in-call ms "
              f"[set/commit+stage, step, get/fetch] {np.median(ts, 0).round(3).tolist()} max {ts.max(0).round(3).tolist()}",
              flush=True)
