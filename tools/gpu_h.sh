mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_h.log 2>&1; echo rc=$? >> gpurun_out/pytest_h.log
timeout 300 python tools/kbench.py --workload cfg2 --algos tc_pipe --iters 20 >> gpurun_out/kbench_h.log 2>&1
for kb in 16 24 32 48 64; do for st in 2 3 4 6 8 12; do
  echo "stage_kb=$kb max_stages=$st" >> gpurun_out/kbench_h.log
  ITLUMM_ENC_STAGE_KB=$kb ITLUMM_ENC_MAX_STAGES=$st timeout 120 python tools/kbench.py --workload cfg2 --algos tc_pipe --only encode --iters 20 >> gpurun_out/kbench_h.log 2>&1
done; done
