VARIANTS="ynorm500" bash tools/variant_multi.sh
SO=paper_1905_10574_b200/librsylv_b200.so; cp $SO /tmp/b6.so
cp build/var/ynorm500_prof.so $SO; python tools/phase_prof.py c5 > gpurun_out/e11_phase.log 2>&1
cp /tmp/b6.so $SO
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pt_ynorm500.log 2>&1; echo rc=$? >> gpurun_out/pt_ynorm500.log
