# round evidence: default bench line, reference arm, launch list, k_persistent traffic, ncu captures
set -x
mkdir -p gpurun_out/ev
python bench.py > gpurun_out/ev/bench_full.json 2> gpurun_out/ev/bench_full.err
python bench.py --impl reference > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err
for c in c1 c2 c3 c4; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e; done > gpurun_out/ev/bench_configs.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_bench_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev/ncu_launch.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum --clock-control none -k regex:k_persistent -c 1 --csv --log-file gpurun_out/ev/traffic_c5_k_persistent.csv python tools/dag_once.py c5 > gpurun_out/ev/ncu_traffic.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_persistent -c 1 -o gpurun_out/ev/prof_c2_persistent python tools/dag_once.py c2 > gpurun_out/ev/ncu_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_update_bench -c 1 -o gpurun_out/ev/prof_update_only_c5 python tools/update_bench.py c5 > gpurun_out/ev/ncu_ub.log 2>&1
