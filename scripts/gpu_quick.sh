#!/bin/bash
# usage: scripts/gpu_quick.sh <tag> [pytest -k expr] — gpu tests, a short bench, the launch list
TAG=${1:-q}
K=${2:-}
cd "$GRAFT_REPO_ROOT" || cd /root/repo
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short -rf -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1
else
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short -rf > gpurun_out/${TAG}_pytest.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > /dev/null 2>&1
tail -2 gpurun_out/${TAG}_pytest.log
