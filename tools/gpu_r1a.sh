#!/bin/bash
# Round-1 GPU pass: parity tests, per-kernel timings, bench line, launch list, one ncu --set full capture.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for w in cfg2 cfg1 cfg3_c64 cfg3_c128 cfg5; do timeout 300 python tools/kbench.py --workload $w --algos simt,tc,tc_pipe --iters 20 >> gpurun_out/kbench.log 2>&1; done
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$? >> gpurun_out/bench.err
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo rc=$? >> gpurun_out/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tc|k_lut|k_encode' -s 6 -c 4 -o gpurun_out/prof_cfg2 $CMD > gpurun_out/ncu_full.log 2>&1
echo rc=$? >> gpurun_out/ncu_full.log
