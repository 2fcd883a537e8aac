#!/bin/bash
# usage: scripts/gpu_pers_ab.sh VARIANT... — ms/step of the small, sweep-heavy configs (persistent /
# cluster PPE loops) for libsisph.so and each libsisph_<VARIANT>.so
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for V in base "$@"; do
  if [ "$V" = base ]; then unset SISPH_LIB; else export SISPH_LIB=$PWD/paper_1908_01762_b200/libsisph_$V.so; fi
  for W in hydrostatic dambreak2d tgv2d; do
    for rep in 1 2; do
      timeout 600 python bench.py --workload $W --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/pers_ab.json 2> gpurun_out/pers_ab.err
      echo "$V $W $(python -c "import json;d=json.load(open('gpurun_out/pers_ab.json'));print(round(d['ms_per_step'],4), d.get('sweeps_per_step'))" 2>&1 | tail -1)"
    done
  done
done
