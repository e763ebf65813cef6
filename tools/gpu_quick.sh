mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_split_packed.py -q -m gpu --timeout 120 -x -k "tc" > gpurun_out/i2f_tests.txt 2>&1; tail -1 gpurun_out/i2f_tests.txt
for i in 1 2; do for w in cfg2 cfg5; do timeout 300 python tools/kbench.py --workload $w --algos tc --only acc --iters 30 >> gpurun_out/quick.txt; done; done
for w in cfg2 cfg2_packed; do timeout 300 python bench.py --workload $w --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$w', round(d['ms_per_step']*1e3,2))" >> gpurun_out/quick.txt; done
