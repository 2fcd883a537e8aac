#!/bin/bash
# usage: scripts/gpu_final.sh <tag> — the round's measurement set: bench (default and reference arm),
# smoke, launch list and ncu --set full captures of the hot kernels (outputs in gpurun_out/)
TAG=${1:-f}
cd "$GRAFT_REPO_ROOT" || cd /root/repo
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
EXTRA_NCU="rhs:k_rhs_diag:0 density:k_density:0 pgrad:k_pgrad_correct:0" bash scripts/gpu_ncu.sh ${TAG}
echo done
