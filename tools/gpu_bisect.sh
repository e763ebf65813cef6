# developer: per-kernel sequence of whole-MLP forwards (kprof) + cfg2 bench + encoder parity tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "tc_pipe or simt" --timeout 300 > gpurun_out/enc_tests.txt 2>&1; tail -1 gpurun_out/enc_tests.txt
for w in cfg4_c256 cfg4_c16; do timeout 600 python tools/kprof.py $w --iters 2 >> gpurun_out/kprof.jsonl 2>>gpurun_out/kprof.err; done
timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('cfg2', d['ms_per_step']*1e3)" >> gpurun_out/kprof.jsonl
