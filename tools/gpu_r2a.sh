#!/bin/bash
# Round 2, call A: baseline of the streamed-LUT k_tc at cfg5 (bench line + ncu --set full of one launch).
mkdir -p gpurun_out/r2a
nvidia-smi -L > gpurun_out/r2a/gpu.txt 2>&1
timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2a/bench_cfg5.json 2> gpurun_out/r2a/bench_cfg5.err
CMD="python tools/kbench.py --workload cfg5 --algos tc --only acc --iters 2 --no-graph"
timeout 600 $CMD > gpurun_out/r2a/kbench_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc -s 3 -c 1 -o gpurun_out/r2a/cfg5_ktc $CMD > gpurun_out/r2a/ncu.log 2>&1
echo rc=$? >> gpurun_out/r2a/ncu.log
