# ring-depth / slice-width sensitivity of the fused k_tc on split-packed cfg2 rows (TMA-staged)
mkdir -p gpurun_out
out=gpurun_out/fusedpk2.txt
: > $out
timeout 300 python -m pytest tests/test_split_packed.py -q -m gpu --timeout 300 -k fused > gpurun_out/fusedpk2_tests.txt 2>&1; tail -1 gpurun_out/fusedpk2_tests.txt >> $out
kb() { echo "$1" >> $out; env $1 timeout 300 python tools/kbench.py --workload cfg2 --packed --algos $2 --only fused --iters 200 >> $out 2>&1; }
for i in 1 2; do
kb "X=0" tc,tc_pipe
kb "ITLUMM_TC_STAGES=2" tc
kb "ITLUMM_TC_NS_MAX=128 ITLUMM_TC_STAGES=6" tc
kb "ITLUMM_TC_NS_MAX=128 ITLUMM_TC_STAGES=4" tc
kb "ITLUMM_TC_NS_MAX=128 ITLUMM_TC_STAGES=6" tc_pipe
done
