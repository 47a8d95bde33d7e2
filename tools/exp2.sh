SO=paper_1905_10574_b200/librsylv_b200.so
cp $SO /tmp/base.so
cp build/var/profile.so $SO; python tools/phase_prof.py c5 c2 > gpurun_out/e2_phase.log 2>&1
cp /tmp/base.so $SO
