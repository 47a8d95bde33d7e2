cat gpurun_out/sb.log; tail -3 gpurun_out/pt.log; grep -E "^(FAILED|E )" gpurun_out/pt.log | head -10
python - << 'PY'
import json
for l in open("gpurun_out/bench.log"):
    if l.startswith("{"):
        d = json.loads(l); print(d["config"]["workload"][:3], round(d["value"]), round(d["ms_per_step"], 2), round(d["roofline"]["frac"], 4))
    else: print(l.rstrip()[:200])
PY
