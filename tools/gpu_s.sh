mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_s.log 2>&1; echo rc=$? >> gpurun_out/pytest_s.log
for w in cfg2 cfg3_c64 cfg3_c128; do for sb in 0 1; do echo "stream=$sb" >> gpurun_out/kbench_s.log; ITLUMM_TC_STREAM=$sb timeout 300 python tools/kbench.py --workload $w --algos tc_pipe --iters 20 >> gpurun_out/kbench_s.log 2>&1; done; done
timeout 300 python tools/kbench.py --workload cfg5 --algos tc_pipe --iters 5 >> gpurun_out/kbench_s.log 2>&1
