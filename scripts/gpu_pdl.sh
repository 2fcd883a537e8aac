#!/bin/bash
# A/B of programmatic dependent launch in the PPE loop (SISPH_PDL=0/1) on the small configs + loop-form tests
cd "$GRAFT_REPO_ROOT" || cd /root/repo
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short -rf -k "loop_forms or sweep_codes or stored" > gpurun_out/pdl_pytest.log 2>&1
tail -3 gpurun_out/pdl_pytest.log
for W in "tgv2d --ppe-loop 2" "tgv2d --ppe-loop 1" "hydrostatic" "hydrostatic --ppe-loop 1" "dambreak2d" "tgv3d"; do
  for s in 0 1; do
    SISPH_PDL=$s timeout 600 python bench.py --workload $W --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/pdl.json 2> gpurun_out/pdl.err
    echo "$W pdl=$s $(python -c "import json;d=json.load(open('gpurun_out/pdl.json'));print(d['ms_per_step'], d.get('sweeps_per_step'))" 2>&1 | tail -1)"
  done
done
