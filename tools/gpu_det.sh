# development: bitwise repeatability of build variants (tools/det_stress.py)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/det.log
for v in "" ${VARIANTS}; do
  make -B -s -C paper_1905_10574_b200/csrc EXTRA="$(echo $v | tr ',' ' ')" > /dev/null 2>&1
  echo "== variant [$v]" >> gpurun_out/det.log
  timeout 900 python tools/det_stress.py ${DETARGS:-c5 0 10} >> gpurun_out/det.log 2>&1
done
