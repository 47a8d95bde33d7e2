# round evidence on HEAD: full GPU suite + bench lines (gpu_suite.sh), then launch list, DRAM traffic and ncu captures (evidence.sh),
# plus the source-level counters of one full c5 DAG
bash tools/gpu_suite.sh
bash tools/evidence.sh > gpurun_out/evidence.log 2>&1
cd $GRAFT_REPO_ROOT
timeout 1500 ncu --section SourceCounters --section WarpStateStats --section SchedulerStats --section ComputeWorkloadAnalysis --section InstructionStats --import-source on --clock-control none -k regex:k_persistent -c 1 -o gpurun_out/ev/prof_c5_dag_source python tools/dag_once.py c5 > gpurun_out/ev/ncu_c5_dag.log 2>&1
