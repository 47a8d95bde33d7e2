# GPU parity evidence: GEMM/residual tests, per-tile + elementwise twin parity (reports in
# gpurun_out/parity_twins.jsonl), literal configs with the full device residual
# (gpurun_out/fullsize_residuals.jsonl)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/parity_twins.jsonl gpurun_out/fullsize_residuals.jsonl
timeout 1500 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity_twins.py tests/test_gpu_fullsize.py -q ${PYTEST_ARGS:-} > gpurun_out/pt_parity.log 2>&1; echo "rc=$?" >> gpurun_out/pt_parity.log
