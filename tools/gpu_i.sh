mkdir -p gpurun_out
timeout 300 python tools/kbench.py --workload cfg2 --algos tc_pipe --iters 20 > gpurun_out/kbench_i.log 2>&1
CMD="python tools/kbench.py --workload cfg2 --algos tc --only acc --iters 3 --no-graph"
timeout 300 $CMD > gpurun_out/plain_i.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tc' -s 2 -c 1 -o gpurun_out/prof_i $CMD > gpurun_out/ncu_i.log 2>&1
echo rc=$? >> gpurun_out/ncu_i.log
