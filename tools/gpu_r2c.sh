#!/bin/bash
# Round 2, call C: first run of the CTA-pair sparse kernel: smoke, small parity, then timing.
mkdir -p gpurun_out/r2c
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c/smoke.log 2>&1; echo rc=$? >> gpurun_out/r2c/smoke.log
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "parity_small" --timeout 300 > gpurun_out/r2c/pytest_small.log 2>&1; echo rc=$? >> gpurun_out/r2c/pytest_small.log
for w in cfg5 cfg3_c128 cfg3_c64; do timeout 300 python tools/kbench.py --workload $w --algos tc,tc_dense,tc_sp24 --only acc --iters 20 >> gpurun_out/r2c/kbench.jsonl 2>> gpurun_out/r2c/kbench.err; done
for w in cfg5 cfg3_c128; do ITLUMM_PAIR=0 timeout 300 python tools/kbench.py --workload $w --algos tc,tc_sp24 --only acc --iters 20 >> gpurun_out/r2c/kbench_pair0.jsonl 2>> gpurun_out/r2c/kbench.err; done
