mkdir -p gpurun_out
for cfg in "24 100" "16 100" "32 100" "24 80" "24 130" "24 160" "32 128" "48 144"; do set -- $cfg
  ITLUMM_ENC_STAGE_KB=$1 ITLUMM_ENC_INFLIGHT_KB=$2 timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('stage=$1 infl=$2', round(d['ms_per_step']*1e3,2))" >> gpurun_out/quick.txt
done
