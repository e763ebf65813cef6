#!/bin/bash
# Round-end evidence (part 2): one ncu --set full capture of the bench step's kernels (after the
# same command exits 0 without ncu).
mkdir -p gpurun_out/final
CMD="python bench.py --steps 20 --warmup 3 --e2e-steps 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/final/plain_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tc|k_encode_rows' -s 6 -c 2 -o gpurun_out/final/prof_cfg2 $CMD > gpurun_out/final/ncu_full.log 2>&1
echo rc=$? >> gpurun_out/final/ncu_full.log
