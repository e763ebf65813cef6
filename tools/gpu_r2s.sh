#!/bin/bash
mkdir -p gpurun_out/r2s
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "parity_small and (9-4097 or 10-3000 or 14-700 or 5-2049)" > gpurun_out/r2s/pytest.log 2>&1
for d in 0 256 64 1; do echo "dbg=$d" >> gpurun_out/r2s/kb.txt; ITLUMM_TCP_DBG=$d timeout 300 python tools/kbench.py --workload cfg5 --algos tc,tc_dense --only acc --iters 10 >> gpurun_out/r2s/kb.txt 2>&1; done
timeout 300 python tools/kbench.py --workload cfg3_c128 --algos tc,tc_dense --only acc --iters 20 >> gpurun_out/r2s/kb.txt 2>&1
ITLUMM_PAIR=0 timeout 300 python tools/kbench.py --workload cfg5 --algos tc --only acc --iters 10 >> gpurun_out/r2s/kb.txt 2>&1
timeout 300 python tools/tcp_trace.py cfg5 tc > gpurun_out/r2s/trace0.txt 2>&1
