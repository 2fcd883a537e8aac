#!/bin/bash
# A/B of SISPH_SWEEP_CODES on the sweep-heavy small configs (C1 tgv2d, C2 hydrostatic, C3 dambreak2d)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for W in tgv2d hydrostatic dambreak2d; do
  for s in 0 1; do
    SISPH_SWEEP_CODES=$s timeout 600 python bench.py --workload $W --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/codess_${W}_$s.json 2> gpurun_out/codess_${W}_$s.err
    echo "$W codes=$s $(python -c "import json;d=json.load(open('gpurun_out/codess_${W}_$s.json'));print(d['ms_per_step'], d['roofline']['frac'], d.get('sweeps_per_step'))")"
  done
done
