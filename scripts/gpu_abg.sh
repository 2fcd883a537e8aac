#!/bin/bash
# A/B: libsisph.so vs libsisph_g1.so (SISPH_LIB), interleaved, 2 rounds
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for r in 1 2; do
for V in base g1; do
  if [ "$V" = base ]; then unset SISPH_LIB; else export SISPH_LIB=$PWD/paper_1908_01762_b200/libsisph_$V.so; fi
  for W in "hydrostatic --ppe-loop 3" "hydrostatic --ppe-loop 2" "dambreak3d" "tgv3d"; do
    timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abg.json 2> gpurun_out/abg.err
    echo "$V $W $(python -c "import json;d=json.load(open('gpurun_out/abg.json'));print(round(d['ms_per_step'],4), d.get('sweeps_per_step'), round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
  done
done
done
