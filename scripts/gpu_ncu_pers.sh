#!/bin/bash
# ncu --set full of the persistent PPE loop kernel on C2 (hydrostatic): one solve
cd "$GRAFT_REPO_ROOT" || cd /root/repo
CMD="python bench.py --workload hydrostatic --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/pers_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_ppe_persistent" -s 3 -c 1 -o gpurun_out/pers $CMD > gpurun_out/pers_ncu.log 2>&1
ncu -i gpurun_out/pers.ncu-rep --page details --csv > gpurun_out/pers_details.csv 2>&1
ncu -i gpurun_out/pers.ncu-rep --page source --csv > gpurun_out/pers_source.csv 2>&1
ls -la gpurun_out/pers*
