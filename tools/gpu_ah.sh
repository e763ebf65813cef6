mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x --timeout 240 > gpurun_out/pytest_ah.log 2>&1; echo rc=$? >> gpurun_out/pytest_ah.log
for w in cfg2 cfg3_c64; do timeout 300 python tools/kbench.py --workload $w --algos simt --summation avg16 --iters 10 >> gpurun_out/kbench_ah.log 2>&1; timeout 300 python tools/kbench.py --workload $w --algos simt --iters 10 >> gpurun_out/kbench_ah.log 2>&1; done
