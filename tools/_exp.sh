cd $GRAFT_REPO_ROOT
make -B -s -C paper_1905_10574_b200/csrc EXTRA="-DRSYLV_FAST_DIAG_BUILD=1" > gpurun_out/exp_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fast_diag" > gpurun_out/exp_pt.log 2>&1; echo "rc=$?" >> gpurun_out/exp_pt.log
for c in c1 c2 c5; do echo "$(RSYLV_B200_FAST_DIAG=1 timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | grep -o '"value": [0-9.]*\|Error.*')  fast $c"; done > gpurun_out/exp_bench.log 2>&1
for c in c1 c2; do echo "$(timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | grep -o '"value": [0-9.]*')  exact $c"; done >> gpurun_out/exp_bench.log 2>&1
make -B -s -C paper_1905_10574_b200/csrc PROFILE=1 EXTRA="-DRSYLV_FAST_DIAG_BUILD=1" > /dev/null 2>&1
RSYLV_B200_FAST_DIAG=1 timeout 300 python tools/phase_prof.py c1 c2 2>&1 | grep -E "fast path per|fast diagonal|dag_ms" > gpurun_out/exp_phase.log 2>&1
