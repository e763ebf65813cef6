mkdir -p gpurun_out
run() { env $2 timeout 600 python bench.py --workload $1 --steps ${3:-10} --warmup 3 --no-cpu-baseline --e2e-steps 2 > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));print(json.dumps({'wl':'$1','env':'$2','us':d['ms_per_step']*1e3,'clk':d['clocks']}))" >> gpurun_out/ab.jsonl; }
for e in "X=0" "ITLUMM_A_HINT=0" "ITLUMM_ENC_PDL=0" "ITLUMM_A_HINT=0 ITLUMM_ENC_PDL=0" "X=0"; do run cfg4_c256 "$e"; done
for e in "X=0" "ITLUMM_A_HINT=0" "X=0"; do run cfg5 "$e" 20; done
