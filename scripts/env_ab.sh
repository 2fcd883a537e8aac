#!/bin/bash
# usage: scripts/env_ab.sh VAR KERNEL_REGEX — bit-identity check + bench + per-kernel times with VAR=0 vs 1
VAR=$1; RE=${2:-k_}
cd "$GRAFT_REPO_ROOT" || cd /root/repo
python scripts/env_ab_check.py $VAR
for s in 0 1; do
  env $VAR=$s python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/envab_$s.json 2>/dev/null
  env $VAR=$s ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$RE" -c 60 --csv --log-file gpurun_out/envab_$s.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  echo "$VAR=$s ms/step $(python -c "import json;print(json.load(open('gpurun_out/envab_$s.json'))['ms_per_step'])")"
  python scripts/launches.py gpurun_out/envab_$s.csv | head -6
done
