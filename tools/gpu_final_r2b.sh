#!/bin/bash
# Round-2 final evidence in one call: part A (smoke, GPU suite, bench lines of every workload, the
# reference arm) then part B (tools/gpu_evidence.sh: launch list, step traffic, ncu --set full).
bash tools/gpu_final_r2a.sh
bash tools/gpu_evidence.sh final2
tail -2 gpurun_out/final2/smoke.log gpurun_out/final2/pytest_gpu.log; cat gpurun_out/final2/bench_*.json | cut -c1-260
