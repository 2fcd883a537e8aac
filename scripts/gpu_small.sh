#!/bin/bash
# usage: scripts/gpu_small.sh <tag> — the small configs under each PPE loop form + launch lists
TAG=${1:-sm}
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for w in hydrostatic tgv2d; do
  for m in 1 2 3; do
    timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --ppe-loop $m > gpurun_out/${TAG}_${w}_m$m.json 2> gpurun_out/${TAG}_${w}_m$m.err
  done
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_${w}_launches.csv python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
echo done
