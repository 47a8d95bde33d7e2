VARIANTS="ips" bash tools/variant_multi.sh
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pt_ips.log 2>&1; echo rc=$? >> gpurun_out/pt_ips.log
