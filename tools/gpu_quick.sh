mkdir -p gpurun_out
for e in "X=0" "ITLUMM_OUT_HINT=92" "ITLUMM_OUT_HINT=91" "ITLUMM_OUT_HINT=90"; do for w in cfg5 cfg2; do env $e timeout 300 python tools/kbench.py --workload $w --algos tc --only acc --iters 10 | sed "s/^/$e /" >> gpurun_out/quick.txt; done; done
