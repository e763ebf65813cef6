mkdir -p gpurun_out
out=gpurun_out/fusedpk4.txt
: > $out
timeout 300 python -m pytest tests/test_split_packed.py -q -m gpu --timeout 300 -k fused > gpurun_out/fusedpk4_tests.txt 2>&1; tail -1 gpurun_out/fusedpk4_tests.txt >> $out
kb() { echo "$1" >> $out; env $1 timeout 300 python tools/kbench.py --workload cfg2 --packed --algos $2 --only fused --iters 200 >> $out 2>&1; }
for i in 1 2; do
kb "X=0" tc,tc_pipe
kb "ITLUMM_TC_PPF=0" tc
kb "ITLUMM_TC_PPF=1" tc
kb "ITLUMM_TC_PPF=3" tc
done
timeout 300 python tools/tc_trace.py cfg2 fusedpk > gpurun_out/trace_fusedpk_ppf2.txt 2>&1
