SO=paper_1905_10574_b200/librsylv_b200.so; cp $SO /tmp/b4.so
cp build/var/mbpf2_prof.so $SO; python tools/phase_prof.py c5 c2 > gpurun_out/e8_phase_mbpf2.log 2>&1
cp build/var/profile.so $SO; python tools/phase_prof.py c5 c2 > gpurun_out/e8_phase_base.log 2>&1
cp /tmp/b4.so $SO
