#!/bin/bash
# Usage: tools/gpu_check.sh TAG [workloads...]  — GPU parity tests, kernel timings and one bench line.
TAG=${1:-x}; shift
WL=${@:-cfg2}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_$TAG.log
for w in $WL; do timeout 300 python tools/kbench.py --workload $w --algos simt,tc,tc_pipe --iters 20 >> gpurun_out/kbench_$TAG.log 2>&1; done
timeout 600 python bench.py --steps 500 --warmup 20 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo rc=$? >> gpurun_out/bench_$TAG.err
