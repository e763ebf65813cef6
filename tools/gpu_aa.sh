mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_aa.log 2>&1; echo rc=$? >> gpurun_out/pytest_aa.log
for w in cfg2 cfg3_c64 cfg3_c128 cfg5; do timeout 300 python tools/kbench.py --workload $w --algos tc_pipe --iters 10 >> gpurun_out/kbench_aa.log 2>&1; done
python tools/tc_trace.py cfg2 > gpurun_out/tc_trace_cfg2_b.txt 2>&1
