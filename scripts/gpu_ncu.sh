#!/bin/bash
# usage: scripts/gpu_ncu.sh <tag> — plain run, launch list, one ncu --set full capture per hot kernel
TAG=${1:-n}
cd "$GRAFT_REPO_ROOT" || cd /root/repo
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_sweep" -s 2 -c 1 -o gpurun_out/${TAG}_sweep $CMD > gpurun_out/${TAG}_ncu_sweep.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_build_cells" -s 4 -c 1 -o gpurun_out/${TAG}_build $CMD > gpurun_out/${TAG}_ncu_build.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_forces_predict" -s 1 -c 1 -o gpurun_out/${TAG}_forces $CMD > gpurun_out/${TAG}_ncu_forces.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_gtvf_substep" -s 3 -c 1 -o gpurun_out/${TAG}_gtvf $CMD > gpurun_out/${TAG}_ncu_gtvf.log 2>&1
echo done
