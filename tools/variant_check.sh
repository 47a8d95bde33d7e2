# usage: VARIANT=name bash tools/variant_check.sh  -> parity tests + per-config bench on build/var/$VARIANT.so
SO=paper_1905_10574_b200/librsylv_b200.so
cp $SO /tmp/base.so
cp build/var/$VARIANT.so $SO
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/v_${VARIANT}_pt.log 2>&1; echo "rc=$?" >> gpurun_out/v_${VARIANT}_pt.log
for c in ${CONFIGS:-c1 c2 c3 c4 c5}; do timeout 300 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], round(d['value']), round(d['roofline']['frac'],4), d['config']['status'])"; done > gpurun_out/v_${VARIANT}_bench.log 2>&1
cp /tmp/base.so $SO
