#!/bin/bash
# A/B: register-buffered appends (default) vs shared-memory ring appends (build, build + filter)
TAG=${1:-ab}
cd "$GRAFT_REPO_ROOT" || cd /root/repo
SISPH_LIB=$PWD/paper_1908_01762_b200/libsisph_ring2.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "neighbor or rstar or full_step or c5" > gpurun_out/${TAG}_pytest_ring.log 2>&1
for v in A B C; do
  case $v in A) unset SISPH_LIB;; B) export SISPH_LIB=$PWD/paper_1908_01762_b200/libsisph_ring.so;; C) export SISPH_LIB=$PWD/paper_1908_01762_b200/libsisph_ring2.so;; esac
  for w in dambreak3d tgv3d; do
    timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${w}_$v.json 2> gpurun_out/${TAG}_${w}_$v.err
  done
  CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_$v.csv $CMD > /dev/null 2>&1
done
echo done
