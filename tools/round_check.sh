# full GPU check on the box: tests, default bench line, per-config bench lines
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for c in ${CONFIGS:-c1 c2 c3 c4}; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e; done > gpurun_out/bench_cfg.log 2>&1
