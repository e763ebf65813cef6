mkdir -p gpurun_out
for wl in cfg2 cfg3_c64 cfg3_c128 cfg5; do
  timeout 300 python tools/kbench.py --workload $wl --algos tc,tc_sp24,tc_pipe,tc_pipe_sp24 --only acc,fused --iters 20 >> gpurun_out/sp24_kbench.jsonl 2>&1
done
for st in 3 4 5 6; do
  ITLUMM_TC_SP_STAGES=$st timeout 300 python tools/kbench.py --workload cfg5 --algos tc_sp24 --only acc --iters 10 | sed "s/^/st=$st /" >> gpurun_out/sp24_kbench.jsonl 2>&1
done
