mkdir -p gpurun_out
for w in cfg2 cfg3_c64; do timeout 300 python tools/kbench.py --workload $w --algos tc,tc_pipe --iters 20 >> gpurun_out/kbench_g.log 2>&1; timeout 300 python tools/kbench.py --no-graph --workload $w --algos tc,tc_pipe --iters 20 >> gpurun_out/kbench_g.log 2>&1; done
CMD="python tools/kbench.py --workload cfg2 --algos tc_pipe --only fused --iters 3 --no-graph"
timeout 300 $CMD > gpurun_out/plain_g.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tc|k_encode' -s 4 -c 2 -o gpurun_out/prof_g $CMD > gpurun_out/ncu_g.log 2>&1
echo rc=$? >> gpurun_out/ncu_g.log
