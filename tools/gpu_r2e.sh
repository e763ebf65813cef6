#!/bin/bash
mkdir -p gpurun_out/r2e
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "parity_small and (case9 or 9-4097 or 10-3000 or 14-700)" --timeout 300 > gpurun_out/r2e/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2e/pytest.log
for w in cfg5 cfg3_c128 cfg3_c64; do timeout 300 python tools/kbench.py --workload $w --algos tc,tc_dense --only acc --iters 20 >> gpurun_out/r2e/kbench.jsonl 2>> gpurun_out/r2e/kbench.err; done
CMD="python tools/kbench.py --workload cfg3_c128 --algos tc --only acc --iters 2 --no-graph"
timeout 300 $CMD > gpurun_out/r2e/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tcp -s 2 -c 1 -o gpurun_out/r2e/tcp_c128 $CMD > gpurun_out/r2e/ncu.log 2>&1
echo rc=$? >> gpurun_out/r2e/ncu.log
