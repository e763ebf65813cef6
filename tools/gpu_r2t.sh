#!/bin/bash
mkdir -p gpurun_out/r2t
ITLUMM_TCP_DBG=1024 timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "parity_small and (9-4097 or 10-3000 or 14-700 or 5-2049)" > gpurun_out/r2t/pytest.log 2>&1
for d in 0 1024 1; do echo "dbg=$d" >> gpurun_out/r2t/kb.txt; ITLUMM_TCP_DBG=$d timeout 300 python tools/kbench.py --workload cfg5 --algos tc_dense --only acc --iters 10 >> gpurun_out/r2t/kb.txt 2>&1; done
ITLUMM_PAIR=0 timeout 300 python tools/kbench.py --workload cfg5 --algos tc --only acc --iters 10 >> gpurun_out/r2t/kb.txt 2>&1
