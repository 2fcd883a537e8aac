#!/bin/bash
# A/B of the sweep's 16-bit list (SISPH_SWEEP_CODES=0/1): bit identity, bench C5 + C4, kernel times
cd "$GRAFT_REPO_ROOT" || cd /root/repo
timeout 600 python scripts/env_ab_check.py SISPH_SWEEP_CODES > gpurun_out/codes_check.txt 2>&1
echo "check rc=$?" >> gpurun_out/codes_check.txt
for W in dambreak3d tgv3d; do
  for s in 0 1; do
    SISPH_SWEEP_CODES=$s timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/codes_${W}_$s.json 2> gpurun_out/codes_${W}_$s.err
    SISPH_SWEEP_CODES=$s timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_sweep|k_rhs_diag" -c 40 --csv --log-file gpurun_out/codes_${W}_$s.csv python bench.py --workload $W --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  done
done
cat gpurun_out/codes_check.txt
