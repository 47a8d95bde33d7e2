REPS=2 python tools/dag_once.py c5 16000 > gpurun_out/e3_plain.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_persistent -c 1 -o gpurun_out/prof_c5at16k_dag python tools/dag_once.py c5 16000 > gpurun_out/e3_ncu.log 2>&1
