cp build/var/pref.so paper_1905_10574_b200/librsylv_b200.so
python tools/subsolve_bench.py > gpurun_out/sb_pref.log 2>&1
VARIANTS="pref" bash tools/variant_multi.sh
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pt_pref.log 2>&1; echo rc=$? >> gpurun_out/pt_pref.log
