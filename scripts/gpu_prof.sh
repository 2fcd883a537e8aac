#!/bin/bash
# usage: scripts/gpu_prof.sh <tag> — launch list + one ncu --set full capture of k_sweep
TAG=${1:-p}
cd "$GRAFT_REPO_ROOT" || cd /root/repo
python scripts/dbg_normals.py > gpurun_out/${TAG}_dbg.log 2>&1
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu1.log 2>&1
$CMD > gpurun_out/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 4 -c 1 -o gpurun_out/${TAG}_sweep $CMD > gpurun_out/${TAG}_ncu2.log 2>&1
echo done
