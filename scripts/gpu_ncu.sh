#!/bin/bash
# usage: scripts/gpu_ncu.sh <tag> — plain run, launch list, one ncu --set full capture per hot kernel
TAG=${1:-n}
cd "$GRAFT_REPO_ROOT" || cd /root/repo
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
# -s counts launches of the matching kernel: sweep 0 = first sweep of the first step (does work);
# build 0 = the first per-step loose build
for spec in "sweep:k_sweep:0" "build:k_build_loose:0" "filter:k_filter:0" "forces:k_forces_predict:0" "gtvf:k_gtvf_substep:3" ${EXTRA_NCU}; do
  IFS=: read name re skip <<< "$spec"
  ncu --set full --clock-control none --import-source on -k "regex:${re}" -s ${skip} -c 1 -o gpurun_out/${TAG}_${name} $CMD > gpurun_out/${TAG}_ncu_${name}.log 2>&1
done
echo done
