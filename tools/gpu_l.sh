mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_l.log 2>&1; echo rc=$? >> gpurun_out/pytest_l.log
for w in cfg2 cfg3_c64 cfg3_c128 cfg1; do timeout 300 python tools/kbench.py --workload $w --algos tc,tc_pipe --iters 20 >> gpurun_out/kbench_l.log 2>&1; done
