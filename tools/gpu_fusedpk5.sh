mkdir -p gpurun_out
out=gpurun_out/fusedpk5.txt
: > $out
kb() { echo "$1" >> $out; env $1 timeout 300 python tools/kbench.py --workload cfg2 --packed --algos $2 --only fused --iters 200 >> $out 2>&1; }
kb "X=0" tc
kb "ITLUMM_TC_DBG=16" tc
kb "ITLUMM_TC_DBG=32" tc
kb "ITLUMM_TC_DBG=2" tc
ITLUMM_TC_DBG=16 timeout 300 python tools/tc_trace.py cfg2 fusedpk > gpurun_out/trace_fusedpk_dbg16.txt 2>&1
