# usage: scripts/ncu_build_loose.sh TAG VARIANT... — one ncu --set full capture of k_build_loose
# (C5 bench, 5th launch) for libsisph.so ("base") and each libsisph_<VARIANT>.so
TAG=${1:-bl}; shift
cd "$GRAFT_REPO_ROOT" || cd /root/repo
for V in base "$@"; do
  if [ "$V" = base ]; then unset SISPH_LIB; else export SISPH_LIB=$PWD/paper_1908_01762_b200/libsisph_$V.so; fi
  timeout 400 ncu --set full --import-source on --clock-control none -k regex:k_build_loose -s 4 -c 1 \
    -o gpurun_out/${TAG}_$V python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_$V.log 2>&1
  echo "$V rc=$?"
done
