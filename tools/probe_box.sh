#!/bin/bash
# One-shot probe of a GPU box: host CPU/memory, GPU, FP64 peaks (DMMA, DFMA, cuBLAS DGEMM).
mkdir -p gpurun_out
{
nproc; free -g; lscpu | grep -E "Model name|Socket|Core|Thread|Flags" | cut -c1-400
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,memory.total --format=csv
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
SMI=$!
./tools/fp64_peak
python - << 'PY'
import torch, time
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
for _ in range(3): c = a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(5):
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print("cuBLAS DGEMM 8192^3 burst: %.2f TFLOP/s" % (2 * 8192**3 / best / 1e9))
t0 = time.time(); n = 0
e0.record()
while time.time() - t0 < 4: c = a @ b; n += 1
e1.record(); torch.cuda.synchronize()
print("cuBLAS DGEMM 8192^3 sustained 4s: %.2f TFLOP/s" % (2 * 8192**3 * n / e0.elapsed_time(e1) / 1e9))
PY
kill $SMI
} > gpurun_out/probe_box.log 2>&1
cat gpurun_out/probe_box.log
