# development: per-phase counters (profile build on the box)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -B -s -C paper_1905_10574_b200/csrc PROFILE=1 > /dev/null 2>&1
timeout 600 python tools/phase_prof.py ${PCONFIGS:-c2 c5} > gpurun_out/phase.log 2>&1
