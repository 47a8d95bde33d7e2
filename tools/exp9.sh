SO=paper_1905_10574_b200/librsylv_b200.so; cp $SO /tmp/b5.so
cp build/var/rot1_prof.so $SO; python tools/phase_prof.py c5 c2 > gpurun_out/e9_phase_rot1.log 2>&1
cp /tmp/b5.so $SO
