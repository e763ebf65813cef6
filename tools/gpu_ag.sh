mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x --timeout 240 > gpurun_out/pytest_ag.log 2>&1; echo rc=$? >> gpurun_out/pytest_ag.log
timeout 300 python tools/kbench.py --workload cfg2 --algos tc_pipe,tc_sp --iters 20 >> gpurun_out/kbench_ag.log 2>&1
for e in 72 80 88; do echo "E=$e" >> gpurun_out/kbench_ag.log; ITLUMM_SP_ENC_CTAS=$e timeout 120 python tools/kbench.py --workload cfg2 --algos tc_sp --only fused --iters 10 >> gpurun_out/kbench_ag.log 2>&1; done
timeout 300 python tools/tc_trace.py cfg2 sp > gpurun_out/tc_trace_cfg2_sp2.txt 2>&1
