#!/bin/bash
# loop-form tests + ms/step of every loop form on the sweep-heavy configs
cd "$GRAFT_REPO_ROOT" || cd /root/repo
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short -rf -k "loop_forms or sweep_codes or stored" > gpurun_out/loops_pytest.log 2>&1
tail -3 gpurun_out/loops_pytest.log
for W in tgv2d hydrostatic dambreak2d; do
  for m in 1 2 3 4; do
    timeout 600 python bench.py --workload $W --ppe-loop $m --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/loops.json 2> gpurun_out/loops.err
    echo "$W loop=$m $(python -c "import json;d=json.load(open('gpurun_out/loops.json'));print(d['ms_per_step'], d.get('sweeps_per_step'))" 2>&1 | tail -1)"
  done
done
for W in dambreak3d tgv3d; do
  timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/loops.json 2> gpurun_out/loops.err
  echo "$W default $(python -c "import json;d=json.load(open('gpurun_out/loops.json'));print(d['ms_per_step'], d.get('sweeps_per_step'), d['roofline']['frac'])" 2>&1 | tail -1)"
done
