mkdir -p gpurun_out
python tools/bwprobe.py > gpurun_out/bwprobe.json 2>&1
CMD="python tools/kbench.py --workload cfg2 --algos tc_pipe --only fused --iters 3"
timeout 300 $CMD > gpurun_out/plain_c.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tc|k_encode' -s 4 -c 2 -o gpurun_out/prof_c $CMD > gpurun_out/ncu_c.log 2>&1
echo rc=$? >> gpurun_out/ncu_c.log
