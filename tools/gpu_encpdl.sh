mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "tc_pipe or tc_sp or auto" --timeout 300 > gpurun_out/encpdl_tests.txt 2>&1; tail -2 gpurun_out/encpdl_tests.txt
for e in 0 1; do
  ITLUMM_ENC_PDL=$e timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --e2e-steps 2 > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));print(json.dumps({'enc_pdl':$e,'us':d['ms_per_step']*1e3,'value':d['value']}))" >> gpurun_out/encpdl.jsonl
done
for wl in cfg1 cfg3_c64 cfg4_c16; do for e in 0 1; do
  ITLUMM_ENC_PDL=$e timeout 300 python bench.py --workload $wl --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 2 > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));print(json.dumps({'wl':'$wl','enc_pdl':$e,'us':d['ms_per_step']*1e3,'value':d['value']}))" >> gpurun_out/encpdl.jsonl
done; done
