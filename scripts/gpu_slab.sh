#!/bin/bash
# slab path on one GPU: dist parity tests, bench with and without --slab-self, launch list of the slab run
cd "$GRAFT_REPO_ROOT" || cd /root/repo
timeout 900 python -m pytest tests/test_gpu_dist.py -q -p no:cacheprovider --tb=short -x 2>&1 | tail -2
for a in "" "--slab-self"; do
  timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $a 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());p=d.get('ms_per_step_phases');print('$a', round(d['ms_per_step'],3), d['sweeps_per_step'], {k:round(v,3) for k,v in p.items() if k!='note'})"
done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/slab_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --slab-self > /dev/null 2>&1
python scripts/launches.py gpurun_out/slab_launches.csv | head -30
