# full GPU test suite + default bench line + c1 line (with its same-config CPU baseline)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/parity_twins.jsonl gpurun_out/fullsize_residuals.jsonl
lscpu > gpurun_out/lscpu.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/pt_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
