#!/bin/bash
mkdir -p gpurun_out/r2g
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "parity_small" --timeout 300 > gpurun_out/r2g/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2g/pytest.log
for w in cfg5 cfg3_c128 cfg3_c64; do timeout 300 python tools/kbench.py --workload $w --algos tc,tc_dense --only acc --iters 20 >> gpurun_out/r2g/kbench.jsonl 2>> gpurun_out/r2g/kbench.err; done
timeout 300 python tools/tcp_trace.py cfg5 tc > gpurun_out/r2g/trace.txt 2>&1
