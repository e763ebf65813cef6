mkdir -p gpurun_out
out=gpurun_out/fusedpk3.txt
: > $out
timeout 300 python -m pytest tests/test_split_packed.py -q -m gpu --timeout 300 -k fused > gpurun_out/fusedpk3_tests.txt 2>&1; tail -1 gpurun_out/fusedpk3_tests.txt >> $out
kb() { echo "$1" >> $out; env $1 timeout 300 python tools/kbench.py --workload cfg2 --packed --algos $2 --only fused --iters 200 >> $out 2>&1; }
for i in 1 2; do
kb "X=0" tc,tc_pipe
kb "ITLUMM_TC_APF=0" tc
kb "ITLUMM_TC_APF=1" tc
kb "ITLUMM_TC_APF=3" tc
kb "ITLUMM_TC_APF=4" tc
done
ITLUMM_TC_APF=2 timeout 300 python tools/tc_trace.py cfg2 fusedpk > gpurun_out/trace_fusedpk_pf2.txt 2>&1
