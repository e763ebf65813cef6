mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x --timeout 120 > gpurun_out/pytest_am.log 2>&1; echo rc=$? >> gpurun_out/pytest_am.log
for w in cfg3_c64 cfg3_c128 cfg5; do timeout 200 python tools/kbench.py --workload $w --algos tc_pipe --iters 10 >> gpurun_out/kbench_am.log 2>&1; done
