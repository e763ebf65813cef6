# developer sweep: L2 eviction hints on the output stores (ITLUMM_OUT_HINT) and row reads (ITLUMM_A_HINT)
mkdir -p gpurun_out
run() {  # workload a_hint
  ITLUMM_A_HINT=$2 timeout 300 python bench.py --workload $1 --steps ${3:-300} --warmup 10 --no-cpu-baseline --e2e-steps 2 > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));print(json.dumps({'wl':'$1','a_hint':$2,'us':d['ms_per_step']*1e3,'value':d['value']}))" >> gpurun_out/hint_sweep2.jsonl
}
for ah in 0 1 3 4 1 0; do run cfg2 $ah; done
for wl in cfg1 cfg3_c64 cfg3_c128; do for ah in 0 1; do run $wl $ah; done; done
for wl in cfg5 cfg4_c16 cfg4_c64; do for ah in 0 1; do run $wl $ah 20; done; done
