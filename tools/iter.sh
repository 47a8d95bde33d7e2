# development loop on the GPU box: sub-block microbenchmark (section split), GPU tests, benches
make -B -C paper_1905_10574_b200/csrc EXTRA=-DRSYLV_SUBPROF > /dev/null 2>&1
python tools/subsolve_bench.py > gpurun_out/sb.log 2>&1
make -B -C paper_1905_10574_b200/csrc > /dev/null 2>&1
python tools/subsolve_bench.py >> gpurun_out/sb.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1
for c in ${CONFIGS:-c1 c2 c3 c5}; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e; done > gpurun_out/bench.log 2>&1
