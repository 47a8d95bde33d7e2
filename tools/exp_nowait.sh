set -x
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for c in c2 c5; do $B --config $c; done > gpurun_out/exp_base.log 2>&1
make -B -C paper_1905_10574_b200/csrc EXTRA=-DRSYLV_EXPERIMENT_NOWAIT=1 > /dev/null 2>&1
for c in c2 c5; do $B --config $c; done > gpurun_out/exp_nowait.log 2>&1
