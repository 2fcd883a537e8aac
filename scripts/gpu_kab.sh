#!/bin/bash
# usage: scripts/gpu_kab.sh TAG VAR KERNEL_REGEX — bit-identity of engine switch VAR (0 vs 1), per-kernel
# launch times of the C5 bench for both settings, one ncu --set full capture of KERNEL_REGEX with VAR=1
TAG=${1:-kab}; VAR=$2; RE=${3:-k_}
cd "$GRAFT_REPO_ROOT" || cd /root/repo
timeout 600 python scripts/env_ab_check.py $VAR > gpurun_out/${TAG}_check.log 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
for s in 0 1; do
  env $VAR=$s timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_$s.csv $CMD > /dev/null 2>&1
  echo "== $VAR=$s" >> gpurun_out/${TAG}_check.log
  python scripts/launches.py gpurun_out/${TAG}_$s.csv | head -14 >> gpurun_out/${TAG}_check.log
done
env $VAR=1 timeout 400 ncu --set full --import-source on --clock-control none -k regex:"$RE" -s 2 -c 1 -o gpurun_out/${TAG}_ncu $CMD > gpurun_out/${TAG}_ncu.log 2>&1
rm -f gpurun_out/${TAG}_?.csv
cat gpurun_out/${TAG}_check.log
