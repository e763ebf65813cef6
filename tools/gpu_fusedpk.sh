# A/B: fused k_tc on split-packed rows (TMA-staged rows; ITLUMM_TC_ATMA=0: per-thread vector loads)
# vs TC_PIPE (encode + accumulate), kbench fused call
mkdir -p gpurun_out
out=gpurun_out/fusedpk.txt
: > $out
timeout 600 python -m pytest tests/test_split_packed.py -q -m gpu --timeout 300 > gpurun_out/fusedpk_tests.txt 2>&1; tail -3 gpurun_out/fusedpk_tests.txt >> $out
for i in 1 2; do
  timeout 300 python tools/kbench.py --workload cfg2 --packed --algos tc,tc_pipe --only fused --iters 200 >> $out 2>&1
  ITLUMM_TC_ATMA=0 timeout 300 python tools/kbench.py --workload cfg2 --packed --algos tc --only fused --iters 200 >> $out 2>&1
  timeout 300 python tools/kbench.py --workload cfg1 --packed --algos tc,tc_pipe --only fused --iters 200 >> $out 2>&1
done
