#!/bin/bash
# Round-2 evidence: GPU tests + smoke, the default bench line, its ncu launch list, steady-state
# step traffic, and ncu --set full of the cfg5 accumulate (each ncu after the same command ran clean).
O=gpurun_out/final2
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rs > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
bash tools/gpu_evidence.sh final2
