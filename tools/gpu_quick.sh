mkdir -p gpurun_out
for e in "X=0" "ITLUMM_OUT_HINT=85" "X=0" "ITLUMM_OUT_HINT=85"; do for w in cfg2 cfg5; do env $e timeout 300 python tools/kbench.py --workload $w --algos tc --only acc --iters 20 | sed "s/^/$e /" >> gpurun_out/quick.txt; done; done
