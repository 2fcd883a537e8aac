#!/bin/bash
# usage: scripts/ab.sh TAG VARIANT...   — per-kernel launch lists of the C5 bench for libsisph.so
# and each libsisph_<VARIANT>.so (built with build.py --out), summarised by scripts/launches.py
TAG=${1:-ab}; shift
cd "$GRAFT_REPO_ROOT" || cd /root/repo
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
for V in base "$@"; do
  if [ "$V" = base ]; then unset SISPH_LIB; else export SISPH_LIB=$PWD/paper_1908_01762_b200/libsisph_$V.so; fi
  $CMD > gpurun_out/${TAG}_${V}_plain.json 2> gpurun_out/${TAG}_${V}_plain.err
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_${V}.csv $CMD > /dev/null 2>&1
  echo "== $V  ms/step $(python -c "import json;print(json.load(open('gpurun_out/${TAG}_${V}_plain.json'))['ms_per_step'])")"
  python scripts/launches.py gpurun_out/${TAG}_${V}.csv | head -12
done
