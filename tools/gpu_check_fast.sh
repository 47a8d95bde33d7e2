# development check of the diagonal-tile fast path: GPU tests, per-config bench lines,
# phase counters (profile build) with the fast path on and off
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pt2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt2.log; fi
for c in ${CONFIGS:-c1 c2 c5}; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e; done > gpurun_out/bench_fast.jsonl 2> gpurun_out/bench_fast.err
make -B -s -C paper_1905_10574_b200/csrc PROFILE=1 > /dev/null 2>&1
(timeout 300 python tools/phase_prof.py ${PCONFIGS:-c1 c2}; RSYLV_B200_FAST_DIAG=1 timeout 300 python tools/phase_prof.py ${PCONFIGS:-c1 c2}) > gpurun_out/phase.log 2>&1
