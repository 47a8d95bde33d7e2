# development: e2e breakdown over shell-group sizes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/e2e_breakdown.log
for g in ${GROUPS_:-1 2 4 8 16}; do
  echo "== RSYLV_B200_SHELL_GROUP=$g" >> gpurun_out/e2e_breakdown.log
  for c in ${CONFIGS:-c5 c4}; do
    RSYLV_B200_SHELL_GROUP=$g RSYLV_B200_DEBUG_TIMING=1 python tools/e2e_breakdown.py $c 1 2>&1 | grep "host pipeline" | tail -1 >> gpurun_out/e2e_breakdown.log
    RSYLV_B200_SHELL_GROUP=$g python tools/e2e_breakdown.py $c 2 2>&1 | grep "host buffers" | tail -1 | cut -c1-215 >> gpurun_out/e2e_breakdown.log
  done
done
