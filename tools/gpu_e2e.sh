# development: e2e breakdown over pipeline settings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/e2e_breakdown.log
for r in ${RESERVES:-1 2 4 8}; do
  echo "== RSYLV_B200_PIPE_RESERVE=$r" >> gpurun_out/e2e_breakdown.log
  for c in ${CONFIGS:-c5}; do
    RSYLV_B200_PIPE_RESERVE=$r python tools/e2e_breakdown.py $c 2 2>&1 | grep "host buffers" | tail -1 | cut -c1-215 >> gpurun_out/e2e_breakdown.log
  done
done
