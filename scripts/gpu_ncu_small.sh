#!/bin/bash
# ncu --set full of the C2 (hydrostatic) sweep and wall pass
TAG=${1:-ns}
cd "$GRAFT_REPO_ROOT" || cd /root/repo
CMD="python bench.py --workload hydrostatic --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_sweep" -s 20 -c 1 -o gpurun_out/${TAG}_sweep $CMD > gpurun_out/${TAG}_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_ppe_wall" -s 20 -c 1 -o gpurun_out/${TAG}_wall $CMD > gpurun_out/${TAG}_ncu2.log 2>&1
echo done
