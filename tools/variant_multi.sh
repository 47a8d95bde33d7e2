# usage: VARIANTS="a b" bash tools/variant_multi.sh -> parity + bench per variant (build/var/<v>.so)
for V in $VARIANTS; do VARIANT=$V bash tools/variant_check.sh; done
SO=paper_1905_10574_b200/librsylv_b200.so; cp $SO /tmp/base2.so
for V in $VARIANTS; do cp build/var/$V.so $SO; UB_DISTINCT= python tools/update_bench.py c5 > gpurun_out/v_${V}_ub.log 2>&1; done
cp /tmp/base2.so $SO
