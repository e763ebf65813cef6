mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_ab.log 2>&1; echo rc=$? >> gpurun_out/pytest_ab.log
timeout 300 python tools/tc_trace.py cfg2 sp > gpurun_out/tc_trace_cfg2_sp.txt 2>&1
timeout 300 python tools/kbench.py --workload cfg2 --algos tc_pipe,tc_sp --only fused --iters 10 >> gpurun_out/kbench_ab.log 2>&1
