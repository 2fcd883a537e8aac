#!/bin/bash
# usage: scripts/gpu_allbench.sh <tag> — one bench line per BASELINE config (C1-C5) into gpurun_out/
TAG=${1:-ab}
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for w in dambreak3d tgv3d dambreak2d hydrostatic tgv2d; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_${w}.json 2> gpurun_out/${TAG}_${w}.err
  echo "$w rc=$?"
done
