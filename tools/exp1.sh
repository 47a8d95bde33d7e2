# update-phase locality experiment + phase counters (prebuilt variants in build/var)
SO=paper_1905_10574_b200/librsylv_b200.so
cp $SO /tmp/base.so
python tools/update_bench.py c5 > gpurun_out/e1_ub.log 2>&1
cp build/var/ub_distinct.so $SO; UB_DISTINCT=1 python tools/update_bench.py c5 > gpurun_out/e1_ub_distinct.log 2>&1
cp build/var/profile.so $SO; python tools/phase_prof.py c5 c2 c1 > gpurun_out/e1_phase.log 2>&1
cp build/var/nowait.so $SO; for c in c2 c5; do python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e; done > gpurun_out/e1_nowait.log 2>&1
cp /tmp/base.so $SO
