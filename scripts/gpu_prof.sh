#!/bin/bash
# usage: scripts/gpu_prof.sh <tag> <kernel-regex> [count]
#   plain bench run, launch list, then one ncu --set full capture of the kernels matching the regex
TAG=${1:-p}
RE=${2:-k_sweep}
CNT=${3:-1}
cd "$GRAFT_REPO_ROOT" || cd /root/repo
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu1.log 2>&1
$CMD > gpurun_out/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:${RE}" -s 8 -c ${CNT} -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu2.log 2>&1
echo done
