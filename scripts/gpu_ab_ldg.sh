#!/bin/bash
# A/B: streaming (__ldcs, default) vs read-only (__ldg) list loads, per workload
TAG=${1:-ab}
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for w in hydrostatic tgv2d dambreak2d dambreak3d; do
  for v in A B; do
    if [ $v = B ]; then export SISPH_LIB=$PWD/paper_1908_01762_b200/libsisph_ldg.so; else unset SISPH_LIB; fi
    timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${w}_$v.json 2> gpurun_out/${TAG}_${w}_$v.err
  done
done
echo done
