python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1
for c in c1 c2 c3 c5; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e; done > gpurun_out/bench.log 2>&1
python tools/update_bench.py > gpurun_out/ub.log 2>&1
make -B -C paper_1905_10574_b200/csrc PROFILE=1 > /dev/null 2>&1; python tools/phase_prof.py c5 > gpurun_out/phase.log 2>&1
