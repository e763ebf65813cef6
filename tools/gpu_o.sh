mkdir -p gpurun_out
CMD="python tools/kbench.py --workload cfg2 --algos tc_sp --only fused --iters 3 --no-graph"
timeout 300 $CMD > gpurun_out/plain_o.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_amm_sp' -s 2 -c 1 -o gpurun_out/prof_o $CMD > gpurun_out/ncu_o.log 2>&1
echo rc=$? >> gpurun_out/ncu_o.log
