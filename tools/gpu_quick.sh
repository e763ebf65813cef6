mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_split_packed.py -q -m gpu --timeout 120 -x > gpurun_out/early_tests.txt 2>&1; tail -1 gpurun_out/early_tests.txt
timeout 200 python tools/kbench.py --workload cfg2 --packed --algos tc --only encode --iters 50 >> gpurun_out/quick.txt
timeout 200 python tools/kbench.py --workload cfg2 --algos tc --only encode --iters 50 >> gpurun_out/quick.txt
for w in cfg2 cfg2_packed cfg1 cfg3_c64_packed; do timeout 300 python bench.py --workload $w --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$w', round(d['ms_per_step']*1e3,2))" >> gpurun_out/quick.txt; done
