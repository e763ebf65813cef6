mkdir -p gpurun_out
timeout 300 python tools/tc_trace.py cfg2 fusedpk > gpurun_out/trace_fusedpk.txt 2>&1
timeout 300 python tools/tc_trace.py cfg2 acc > gpurun_out/trace_acc.txt 2>&1
