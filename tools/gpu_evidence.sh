#!/bin/bash
# Bench line of the default workload (cfg5) + its evidence: ncu launch list of the same command,
# steady-state DRAM traffic of one call (--cache-control none), ncu --set full of the accumulate.
# Usage: bash tools/gpu_evidence.sh <outdir>
O=gpurun_out/${1:-ev}
mkdir -p $O
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err
CMD="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
timeout 900 $CMD > $O/plain_launch.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg5.csv $CMD > $O/ncu_launch.log 2>&1
echo rc=$? >> $O/ncu_launch.log
CMD2="python tools/step_traffic.py run cfg5"
timeout 600 $CMD2 > $O/plain_traffic.log 2>&1 && \
timeout 900 ncu --cache-control none --clock-control none --print-units base --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file $O/traffic_cfg5.csv $CMD2 > $O/ncu_traffic.log 2>&1
echo rc=$? >> $O/ncu_traffic.log
CMD3="python tools/kbench.py --workload cfg5 --algos tc --only acc --iters 2 --no-graph"
timeout 600 $CMD3 > $O/plain_full.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc -s 3 -c 1 -o $O/cfg5_acc $CMD3 > $O/ncu_full.log 2>&1
echo rc=$? >> $O/ncu_full.log
