mkdir -p gpurun_out
for e in 80 88 96; do for inf in 100 150 190; do echo "E=$e infl=$inf" >> gpurun_out/kbench_ae.log; ITLUMM_SP_ENC_CTAS=$e ITLUMM_SP_INFLIGHT_KB=$inf timeout 120 python tools/kbench.py --workload cfg2 --algos tc_sp --only fused --iters 10 >> gpurun_out/kbench_ae.log 2>&1; done; done
