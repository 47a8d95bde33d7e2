SO=paper_1905_10574_b200/librsylv_b200.so; cp $SO /tmp/b7.so
cp build/var/cur_prof.so $SO; python tools/phase_prof.py c5 > gpurun_out/e12_phase.log 2>&1
for v in cur_nopf cur; do cp build/var/$v.so $SO; for c in c5 c2; do python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['workload'][:3], round(d['value']))"; done; done > gpurun_out/e12_bench.log 2>&1
cp /tmp/b7.so $SO
