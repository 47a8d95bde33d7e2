# development iteration: the fast GPU parity files, the update-only throughput and per-config bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_multirank.py tests/test_gpu_pipeline.py} -m gpu -x -q > gpurun_out/pt_iter.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_iter.log
timeout 300 python tools/update_bench.py c5 > gpurun_out/ub_iter.log 2>&1
for c in ${CONFIGS:-c2 c5}; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e; done > gpurun_out/bench_iter.jsonl 2> gpurun_out/bench_iter.err
