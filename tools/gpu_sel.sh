#!/bin/bash
# Selector-mode bring-up: targeted parity tests, then accumulate/fused timings dense vs selector.
TAG=${1:-sel}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -p no:cacheprovider -x -k "sel or streamed" > gpurun_out/pytest_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_$TAG.log
for w in cfg5 cfg3_c128 cfg3_c64; do
  timeout 300 python tools/kbench.py --workload $w --algos tc_pipe_dense,tc_pipe_sel,tc_pipe_sp24 --only acc,fused --iters 20 >> gpurun_out/kbench_$TAG.log 2>&1
done
