mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for w in cfg2 cfg1 cfg3_c64 cfg3_c128; do timeout 300 python tools/kbench.py --workload $w --algos simt,tc,tc_pipe --iters 20 >> gpurun_out/kbench7.log 2>&1; done
timeout 300 python bench.py --steps 1000 --warmup 20 > gpurun_out/bench7.log 2>&1
