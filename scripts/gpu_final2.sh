#!/bin/bash
# usage: scripts/gpu_final2.sh <tag> — the round's measurement set: smoke, default bench line, the
# reference arm, one bench line per config, launch lists, ncu --set full captures of the hot kernels
# of C5 and of the sweep (+ build) of every other workload (outputs in gpurun_out/)
TAG=${1:-f}
cd "$GRAFT_REPO_ROOT" || cd /root/repo
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
for w in tgv3d dambreak2d hydrostatic tgv2d; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_${w}.json 2> gpurun_out/${TAG}_bench_${w}.err
done
for w in dambreak3d tgv3d dambreak2d hydrostatic tgv2d; do
  CMD="python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/${TAG}_${w}_launches.csv $CMD > /dev/null 2>&1
done
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
for spec in "sweep:k_sweep:0" "build:k_build_loose:0" "filter:k_filter:0" "forces:k_forces_predict:0" "gtvf:k_gtvf_substep:3" "rhs:k_rhs_diag:0" "density:k_density:0" "pgrad:k_pgrad_correct:0"; do
  IFS=: read name re skip <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${re}" -s ${skip} -c 1 -o gpurun_out/${TAG}_dambreak3d_${name} $CMD > gpurun_out/${TAG}_ncu_dambreak3d_${name}.log 2>&1
done
for w in tgv3d dambreak2d hydrostatic tgv2d; do
  CMD="python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
  for spec in "sweep:k_sweep:2" "build:k_build_loose:0"; do
    IFS=: read name re skip <<< "$spec"
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${re}" -s ${skip} -c 1 -o gpurun_out/${TAG}_${w}_${name} $CMD > gpurun_out/${TAG}_ncu_${w}_${name}.log 2>&1
  done
done
# summaries on the box (gpurun copies back at most 64 MiB): keep the C5 sweep and build reports
for w in dambreak3d tgv3d dambreak2d hydrostatic tgv2d; do
  python scripts/ncu_summary.py --workload $w --outdir gpurun_out gpurun_out/${TAG}_ncu_${w}.txt gpurun_out/${TAG}_${w}_*.ncu-rep > /dev/null 2>&1
  python scripts/launches.py gpurun_out/${TAG}_${w}_launches.csv > gpurun_out/${TAG}_${w}_launches.txt 2>/dev/null
done
for r in gpurun_out/${TAG}_*.ncu-rep; do
  case $r in *dambreak3d_sweep*|*dambreak3d_build*) ;; *) rm -f $r;; esac
done
rm -f gpurun_out/${TAG}_*_launches.csv
echo done
