# development: per-phase counters (profile build on the box) and the update-only bench with distinct sources per CTA
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -B -s -C paper_1905_10574_b200/csrc EXTRA=-DRSYLV_UB_DISTINCT=1 > /dev/null 2>&1
UB_DISTINCT=1 timeout 300 python tools/update_bench.py c5 > gpurun_out/ub_distinct.log 2>&1
make -B -s -C paper_1905_10574_b200/csrc PROFILE=1 > /dev/null 2>&1
timeout 600 python tools/phase_prof.py ${PCONFIGS:-c2 c5} > gpurun_out/phase.log 2>&1
