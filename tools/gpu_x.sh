mkdir -p gpurun_out
for cfgs in "256 3" "256 4" "192 3" "192 4" "128 4" "128 6"; do set -- $cfgs; echo "ns=$1 st=$2" >> gpurun_out/kbench_x.log; ITLUMM_TC_NS_MAX=$1 ITLUMM_TC_STAGES=$2 timeout 300 python tools/kbench.py --workload cfg2 --algos tc_pipe --iters 20 >> gpurun_out/kbench_x.log 2>&1; done
for st in 2 3 4 5; do echo "cfg5 st=$st" >> gpurun_out/kbench_x.log; ITLUMM_TC_STAGES=$st timeout 300 python tools/kbench.py --workload cfg5 --algos tc_pipe --only acc --iters 5 >> gpurun_out/kbench_x.log 2>&1; done
