mkdir -p gpurun_out
timeout 120 python tools/kbench.py --workload cfg2 --algos tc --only acc --iters 3 > gpurun_out/plain6a.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_tc -s 2 -c 1 -o gpurun_out/prof_tc_acc_cfg2 python tools/kbench.py --workload cfg2 --algos tc --only acc --iters 3 > gpurun_out/ncu6a.log 2>&1
timeout 120 python tools/kbench.py --workload cfg2 --algos tc --only fused --iters 3 > gpurun_out/plain6b.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_tc -s 2 -c 1 -o gpurun_out/prof_tc_fused_cfg2 python tools/kbench.py --workload cfg2 --algos tc --only fused --iters 3 > gpurun_out/ncu6b.log 2>&1
echo done
