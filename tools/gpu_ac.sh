mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x --timeout 240 > gpurun_out/pytest_ac.log 2>&1; echo rc=$? >> gpurun_out/pytest_ac.log
timeout 300 python tools/tc_trace.py cfg2 sp > gpurun_out/tc_trace_cfg2_sp.txt 2>&1
for w in cfg2 cfg3_c64 cfg5; do timeout 300 python tools/kbench.py --workload $w --algos tc,tc_pipe,tc_sp --iters 10 >> gpurun_out/kbench_ac.log 2>&1; done
