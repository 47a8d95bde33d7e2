VARIANTS="mbpf mbnopf" bash tools/variant_multi.sh
SO=paper_1905_10574_b200/librsylv_b200.so; cp $SO /tmp/b3.so
cp build/var/mbpf_distinct.so $SO; UB_DISTINCT=1 python tools/update_bench.py c5 > gpurun_out/v_mbpf_ubd.log 2>&1
cp /tmp/b3.so $SO
