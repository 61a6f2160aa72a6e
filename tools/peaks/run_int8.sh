#!/bin/bash
# INT8 tensor peaks on the GPU box: legacy mma.sync IMMA and torch._int_mm (cuBLASLt, tcgen05)
set -e
cd "$(dirname "$0")"
mkdir -p ../../gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/int8_peaks int8_peaks.cu
/tmp/int8_peaks > ../../gpurun_out/int8_peaks.json
cuobjdump -sass /tmp/int8_peaks | grep -m3 -o "IMMA[^ ]*" >> ../../gpurun_out/int8_sass.txt || true
python - <<'PY' >> ../../gpurun_out/int8_peaks.json
import torch, json
n = 8192
a = torch.randint(-100, 100, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-100, 100, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
for _ in range(2): torch._int_mm(a, b)
torch.cuda.synchronize()
best = 0
for _ in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); torch._int_mm(a, b); e1.record(); torch.cuda.synchronize()
    best = max(best, 2 * n**3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
print(json.dumps({"torch_int_mm_tops_8192": best}))
PY
cat ../../gpurun_out/int8_peaks.json ../../gpurun_out/int8_sass.txt
