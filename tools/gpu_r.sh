mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_r.log 2>&1; echo rc=$? >> gpurun_out/pytest_r.log
for w in cfg5 cfg3_c128 cfg2; do timeout 600 python tools/kbench.py --workload $w --algos tc,tc_pipe --iters 5 >> gpurun_out/kbench_r.log 2>&1; done
