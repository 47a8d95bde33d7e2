# development: single-warp sub-block solve latency + c2/c4 bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/subsolve_bench.py > gpurun_out/subsolve.log 2>&1
for c in ${CONFIGS:-c2 c4}; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e; done > gpurun_out/bench_iter.jsonl 2> gpurun_out/bench_iter.err
