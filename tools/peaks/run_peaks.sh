#!/bin/bash
# Measure FP64 / on-chip peaks on the GPU box (run under gpurun). Writes gpurun_out/fp64_peaks.json
# and the clocks seen while the microbenchmarks ran.
set -e
cd "$(dirname "$0")"
mkdir -p ../../gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peaks fp64_peaks.cu
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active \
  --format=csv -lms 200 > ../../gpurun_out/peaks_clocks.csv &
SMI=$!
/tmp/fp64_peaks > ../../gpurun_out/fp64_peaks.json
python - <<'EOF' >> ../../gpurun_out/fp64_peaks_torch.json
import torch, time, json
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
for _ in range(2): torch.matmul(a, b)
torch.cuda.synchronize()
best = 0
for _ in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    best = max(best, 2 * 8192**3 / t / 1e12)
print(json.dumps({"dgemm_tflops_8192": best}))
EOF
kill $SMI || true
cat ../../gpurun_out/fp64_peaks.json ../../gpurun_out/fp64_peaks_torch.json
