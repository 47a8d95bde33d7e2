# development: bitwise repeatability (tools/det_stress.py) of the default build (+ variants)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/det.log
for v in ${VARIANTS:-default}; do
  vv=$(echo $v | tr ',' ' '); [ "$v" = "default" ] && vv=""
  make -B -s -C paper_1905_10574_b200/csrc EXTRA="$vv" > /dev/null 2>&1
  echo "== variant [$v]" >> gpurun_out/det.log
  timeout 600 python tools/det_stress.py c5 4096 ${REPS:-100} >> gpurun_out/det.log 2>&1
  timeout 600 python tools/det_stress.py c5 12000 ${REPS:-100} >> gpurun_out/det.log 2>&1
  timeout 600 python tools/det_stress.py c2 6000 ${REPS:-100} >> gpurun_out/det.log 2>&1
  timeout 600 python tools/det_stress.py c3 6000 ${REPS:-100} >> gpurun_out/det.log 2>&1
  timeout 600 python tools/det_stress.py c4 0 40 >> gpurun_out/det.log 2>&1
  timeout 900 python tools/det_stress.py c5 0 16 >> gpurun_out/det.log 2>&1
done
