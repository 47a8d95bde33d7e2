cp build/var/ips2.so paper_1905_10574_b200/librsylv_b200.so
VARIANTS="ips2" bash tools/variant_multi.sh
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pt_ips2.log 2>&1; echo rc=$? >> gpurun_out/pt_ips2.log
