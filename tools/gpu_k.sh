mkdir -p gpurun_out
for ns in 64 128 256; do echo "ns_max=$ns" >> gpurun_out/kbench_k.log; ITLUMM_TC_NS_MAX=$ns timeout 300 python tools/kbench.py --workload cfg2 --algos tc_pipe --iters 20 >> gpurun_out/kbench_k.log 2>&1;  ITLUMM_TC_NS_MAX=$ns timeout 300 python tools/kbench.py --workload cfg3_c64 --algos tc_pipe --iters 20 >> gpurun_out/kbench_k.log 2>&1; done
