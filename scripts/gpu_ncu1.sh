#!/bin/bash
# usage: scripts/gpu_ncu1.sh <tag> <kernel-regex> [skip] — one ncu --set full capture (with source) of one kernel
TAG=$1; RE=$2; SKIP=${3:-0}
cd "$GRAFT_REPO_ROOT" || cd /root/repo
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/${TAG}_plain.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${RE}" -s ${SKIP} -c 1 -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo done
