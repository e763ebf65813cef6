mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_split_packed.py -q -m gpu --timeout 120 -x > gpurun_out/ring_tests.txt 2>&1; tail -1 gpurun_out/ring_tests.txt
for e in "ITLUMM_TC_STAGES=4 ITLUMM_TC_BSTAGES=4" "X=0" "ITLUMM_TC_STAGES=5 ITLUMM_TC_BSTAGES=3" "ITLUMM_TC_STAGES=4 ITLUMM_TC_BSTAGES=3" "ITLUMM_TC_STAGES=6 ITLUMM_TC_BSTAGES=2"; do for w in cfg3_c128 cfg5; do env $e timeout 300 python tools/kbench.py --workload $w --algos tc --only acc --iters 10 | sed "s/^/$e /" >> gpurun_out/quick.txt; done; done
