# development: selected GPU test files + one bench config
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -q > gpurun_out/pt_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_quick.log
for c in ${CONFIGS:-}; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e; done > gpurun_out/bench_quick.jsonl 2> gpurun_out/bench_quick.err
