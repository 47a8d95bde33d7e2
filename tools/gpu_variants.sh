# development: c5 DAG time of timing-only build variants (results of the variants are garbage)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/variants.log
for v in "" ${VARIANTS}; do
  make -B -s -C paper_1905_10574_b200/csrc EXTRA="$(echo $v | tr ',' ' ')" > /dev/null 2>&1
  echo "== variant [$v]" >> gpurun_out/variants.log
  for c in ${CONFIGS:-c5}; do timeout 300 python tools/dag_once.py $c >> gpurun_out/variants.log 2>&1; done
done
