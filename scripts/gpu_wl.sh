#!/bin/bash
# usage: scripts/gpu_wl.sh TAG "PYTEST_K" WORKLOAD... — selected GPU tests, then per workload a short bench
# line and the per-kernel launch list (ncu gpu__time_duration, summarised)
TAG=${1:-wl}; K=$2; shift 2
cd "$GRAFT_REPO_ROOT" || cd /root/repo
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short -rf -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
  tail -3 gpurun_out/${TAG}_pytest.log
fi
for w in "$@"; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${w}.json 2> gpurun_out/${TAG}_${w}.err
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_${w}.json').read().strip().splitlines()[-1]);print('$w ms/step', round(d['ms_per_step'],3), 'sweeps', d.get('sweeps_per_step'), 'frac', round(d['roofline']['frac'],3))"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_${w}.csv python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python scripts/launches.py gpurun_out/${TAG}_${w}.csv | head -16
  rm -f gpurun_out/${TAG}_${w}.csv
done
