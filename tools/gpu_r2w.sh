#!/bin/bash
mkdir -p gpurun_out/r2w
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "parity_small or edge or cfg1 or cfg2" > gpurun_out/r2w/pytest.log 2>&1
for w in cfg5 cfg3_c128 cfg3_c64 cfg2; do ITLUMM_PAIR=0 timeout 300 python tools/kbench.py --workload $w --algos tc --only acc --iters 20 >> gpurun_out/r2w/kb_1cta.txt 2>&1; timeout 300 python tools/kbench.py --workload $w --algos tc,tc_dense --only acc --iters 20 >> gpurun_out/r2w/kb_pair.txt 2>&1; done
for w in cfg2 cfg2_packed; do timeout 300 python bench.py --workload $w --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2w/bench_$w.json 2> gpurun_out/r2w/bench_$w.err; done
