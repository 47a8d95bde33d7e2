SO=paper_1905_10574_b200/librsylv_b200.so; cp $SO /tmp/b5.so
cp build/var/rot1_prof_nops.so $SO; python tools/phase_prof.py c5 > gpurun_out/e10_phase_nops.log 2>&1
cp /tmp/b5.so $SO
